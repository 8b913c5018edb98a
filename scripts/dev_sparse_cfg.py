import sys, time; sys.path.insert(0, '.')
import numpy as np, scipy.sparse as sp
import __graft_entry__ as g; g.build()
import paper_1910_01312_b200 as P
from paper_1910_01312_b200 import datagen
k = int(sys.argv[1]); n = int(sys.argv[2]); q = int(sys.argv[3])
t = time.time()
cfg = datagen.make_config(k, n=n, q=q)
print('gen', time.time() - t, flush=True)
A = (cfg['indptr'], cfg['indices'], cfg['data'], cfg['shape'])
pb = P.build_csvc_dual(A, cfg['y'], cfg['C'])
rows = []
t = time.time()
r = P.alm_solve(pb, P.AlmOptions(tol_kkt=1e-6, max_outer=12), P.SsnOptions(cg_max_iters=int(sys.argv[4]) if len(sys.argv) > 4 else 500, eta=float(sys.argv[5]) if len(sys.argv) > 5 else 1e-2), callback=lambda *a: rows.append(a))
print('solve', time.time() - t, r.converged, r.kkt_residual, r.outer_iters, r.total_inner_iters, pb.native_counters)
for row in rows: print('   ', row)
