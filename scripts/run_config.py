"""Solve one BASELINE config with the product path and print a JSON summary."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import __graft_entry__ as g

g.build()
import paper_1910_01312_b200 as P
from paper_1910_01312_b200 import datagen

k = int(sys.argv[1])
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
kw = {}
if scale != 1.0:
    base = {0: (2000, 50), 1: (50000, 300), 4: (1_000_000, 500)}[k]
    kw = {"n": int(base[0] * scale), "q": base[1]}
t0 = time.time()
cfg = datagen.make_config(k, **kw)
tgen = time.time() - t0
if "indptr" in cfg:
    pb = P.build_csvc_dual((cfg["indptr"], cfg["indices"], cfg["data"], cfg["shape"]), cfg["y"],
                           cfg["C"])
elif cfg["task"] == "csvc":
    pb = P.build_csvc_dual(cfg["A"], cfg["y"], cfg["C"])
else:
    pb = P.build_svr_dual(cfg["A"], cfg["t"], cfg["C"], cfg["epsilon"])
rows = []
out = {}
# the large sparse configs need more inner Newton steps than the reference default 50
# at sigma >= 3125
so = datagen.solve_options(cfg)
ssn = P.SsnOptions(**so["ssn"])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
for rep_i in range(reps):
    torch.cuda.synchronize()
    t0 = time.time()
    r = P.alm_solve(pb, P.AlmOptions(tol_kkt=1e-6, **so["alm"]), ssn,
                    callback=(lambda *a: rows.append(a)) if rep_i == 0 else None)
    torch.cuda.synchronize()
    out[f"solve{rep_i}_s"] = time.time() - t0
x = r.x_opt
box_ok = bool(x.min() >= -1e-12 and x.max() <= cfg["C"] + 1e-12)
out.update({"config": k, "n": pb.n, "q": pb.q_op.q, "gen_s": tgen, "kkt": r.kkt_residual,
            "objective": r.objective, "outer": r.outer_iters, "inner": r.total_inner_iters,
            "p": r.unbounded_support_count, "converged": r.converged, "box_ok": box_ok,
            "warnings": r.warnings, "trace": rows, "ssn_options": {"max_inner": ssn.max_inner, "psi_eval": ssn.psi_eval}, "alm_options": so["alm"], "counters": getattr(pb, "native_counters", None)})
print(json.dumps(out))
