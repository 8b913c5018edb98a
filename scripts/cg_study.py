"""Sparse-CG knobs on config 3 at 1/10 scale (n=400k, q=100k, Zipf): time, Newton steps and
CG iterations for each SSNAL_CG_ETA_CAP / SSNAL_CG_BATCH setting (one process per setting)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "run":
    sys.path.insert(0, ROOT)
    import time

    import torch

    import __graft_entry__ as g

    g.build()
    import paper_1910_01312_b200 as P
    from paper_1910_01312_b200 import datagen

    n, q = int(sys.argv[2]), int(sys.argv[3])
    cfg = datagen.config3(n=n, q=q)
    pb = P.build_csvc_dual((cfg["indptr"], cfg["indices"], cfg["data"], cfg["shape"]), cfg["y"],
                           cfg["C"])
    out = {}
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.time()
        r = P.alm_solve(pb, P.AlmOptions(tol_kkt=1e-6), P.SsnOptions(max_inner=200))
        torch.cuda.synchronize()
        out[f"t{rep}"] = time.time() - t0
    out.update(kkt=r.kkt_residual, obj=r.objective, outer=r.outer_iters,
               inner=r.total_inner_iters, converged=r.converged, **pb.native_counters)
    print(json.dumps(out))
    sys.exit(0)

n, q = (sys.argv[1], sys.argv[2]) if len(sys.argv) > 2 else ("400000", "100000")
for cap in ("1e-4", "1e-3", "1e-2"):
    for batch in ("16", "8"):
        env = dict(os.environ, SSNAL_CG_ETA_CAP=cap, SSNAL_CG_BATCH=batch)
        r = subprocess.run([sys.executable, __file__, "run", n, q], env=env, capture_output=True,
                           text=True, timeout=900)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
        print(f"cap={cap} batch={batch}: {line}", flush=True)
