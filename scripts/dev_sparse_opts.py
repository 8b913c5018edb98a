"""Dev: solve a (scaled) sparse config with option overrides from the command line.
    python scripts/dev_sparse_opts.py K n q key=value ...   (keys: AlmOptions / SsnOptions fields)"""
import sys, time; sys.path.insert(0, '.')
import __graft_entry__ as g; g.build()
import paper_1910_01312_b200 as P
from paper_1910_01312_b200 import datagen
k = int(sys.argv[1]); n = int(sys.argv[2]); q = int(sys.argv[3])
alm, ssn = {"tol_kkt": 1e-6, "max_outer": 30}, {}
for kv in sys.argv[4:]:
    key, val = kv.split("=")
    dflt = getattr(P.AlmOptions() if key in P.AlmOptions.__dataclass_fields__ else P.SsnOptions(), key)
    (alm if key in P.AlmOptions.__dataclass_fields__ else ssn)[key] = (
        val if isinstance(dflt, str) else type(dflt)(float(val)))
t = time.time()
cfg = datagen.make_config(k, n=n, q=q)
A = (cfg['indptr'], cfg['indices'], cfg['data'], cfg['shape'])
pb = P.build_csvc_dual(A, cfg['y'], cfg['C'])
print('gen+build', round(time.time() - t, 2), alm, ssn, flush=True)
t0 = time.time()
r = P.alm_solve(pb, P.AlmOptions(**alm), P.SsnOptions(**ssn),
                callback=lambda *a: print('   ', a, round(time.time() - t0, 2), flush=True))
print('solve', round(time.time() - t0, 2), r.converged, r.kkt_residual, r.objective, r.outer_iters,
      r.total_inner_iters, pb.native_counters, r.warnings, flush=True)
