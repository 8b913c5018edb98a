"""Sparse-config solve for ncu launch windows: python scripts/prof_sparse.py K [max_outer]
(K = 2 or 3; the solve runs with datagen.solve_options: max_inner=200, sigma_max=625)."""
import sys
import time

sys.path.insert(0, ".")
import __graft_entry__ as g

g.build()
import paper_1910_01312_b200 as P
from paper_1910_01312_b200 import datagen

k = int(sys.argv[1])
max_outer = int(sys.argv[2]) if len(sys.argv) > 2 else 100
t0 = time.time()
cfg = datagen.make_config(k)
pb = P.build_csvc_dual((cfg["indptr"], cfg["indices"], cfg["data"], cfg["shape"]), cfg["y"], cfg["C"])
print("gen+build", time.time() - t0, flush=True)
t0 = time.time()
so = datagen.solve_options(cfg)
r = P.alm_solve(pb, P.AlmOptions(tol_kkt=1e-6, max_outer=max_outer, **so["alm"]),
                P.SsnOptions(**so["ssn"]))
print("solve", time.time() - t0, r.converged, r.kkt_residual, r.outer_iters, r.total_inner_iters,
      getattr(pb, "native_counters", None), flush=True)
