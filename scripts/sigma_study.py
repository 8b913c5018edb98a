"""ALM penalty schedule vs CG work on config 3 (scale given): python scripts/sigma_study.py
scale|c2|c4 growth,sigma_max,sigma0 ...; prints per-outer rows and totals per setting."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch

import __graft_entry__ as g

g.build()
import paper_1910_01312_b200 as P
from paper_1910_01312_b200 import datagen

if sys.argv[1] == "c2":  # config 2 at full size
    cfg = datagen.config2()
elif sys.argv[1] == "c4":  # config 4 (dense eps-SVR) at full size
    cfg = datagen.config4()
elif sys.argv[1] == "c1":  # config 1 (dense C-SVC 50,000 x 300)
    cfg = datagen.config1()
else:
    scale = float(sys.argv[1])
    cfg = datagen.config3(n=int(4_000_000 * scale), q=int(1_000_000 * scale))
if cfg["task"] == "svr":
    pb = P.build_svr_dual(cfg["A"], cfg["t"], cfg["C"], cfg["epsilon"])
elif "A" in cfg:
    pb = P.build_csvc_dual(cfg["A"], cfg["y"], cfg["C"])
else:
    pb = P.build_csvc_dual((cfg["indptr"], cfg["indices"], cfg["data"], cfg["shape"]), cfg["y"], cfg["C"])
ssn = P.SsnOptions(**datagen.solve_options(cfg)["ssn"])
for spec in sys.argv[2:]:
    growth, smax, s0 = (float(v) for v in spec.split(","))
    rows = []
    torch.cuda.synchronize()
    t0 = time.time()
    r = P.alm_solve(pb, P.AlmOptions(tol_kkt=1e-6, sigma0=s0, sigma_growth=growth, sigma_max=smax),
                    ssn, callback=lambda *a: rows.append(a))
    torch.cuda.synchronize()
    out = dict(spec=spec, t=time.time() - t0, kkt=r.kkt_residual, obj=r.objective, outer=r.outer_iters,
               inner=r.total_inner_iters, converged=r.converged, cg=pb.native_counters["cg_iters"],
               gram_rows=pb.native_counters.get("gram_rows"),
               trace=[(k, f"{res:.2e}", s, p, i) for k, res, s, p, i in rows])
    print(json.dumps(out), flush=True)
