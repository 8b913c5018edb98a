import sys; sys.path.insert(0, ".")
import __graft_entry__ as g; g.build()
import numpy as np
import paper_1910_01312_b200 as pkg
from paper_1910_01312_b200 import datagen, sharded
cfg = datagen.make_config(4, n=20000, q=50)
A, t = cfg["A"], cfg["t"]
world = 2
cuts = [sharded.shard_range(A.shape[0], r, world) for r in range(world)]
probs = [pkg.build_svr_dual(A[lo:hi], t[lo:hi], cfg["C"], cfg["epsilon"]) for lo, hi in cuts]
try:
    reps = sharded.solve_loopback(probs, pkg.AlmOptions(tol_kkt=1e-6))
    print(reps[0])
except Exception as e:
    print("ERR", e)
