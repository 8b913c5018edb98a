"""Run config-1 solves (first one warms up) for ncu launch lists / captures."""
import sys
sys.path.insert(0, '.')
import numpy as np
import __graft_entry__ as g
g.build()
import paper_1910_01312_b200 as P
from paper_1910_01312_b200 import datagen
cfg = datagen.make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
pb = P.build_csvc_dual(cfg["A"], cfg["y"], cfg["C"])
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    r = P.alm_solve(pb, P.AlmOptions(tol_kkt=1e-6))
    print(i, r.converged, r.kkt_residual, r.outer_iters, r.total_inner_iters, r.wall_time, P.default_backend().launch_count())
