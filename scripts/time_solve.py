"""Median device time of K config-k solves (A resident), for quick A/B runs of kernel variants."""
import sys, statistics
sys.path.insert(0, '.')
import torch
import __graft_entry__ as g
g.build()
import paper_1910_01312_b200 as P
from paper_1910_01312_b200 import datagen
k = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = datagen.make_config(k)
pb = P.build_csvc_dual(cfg["A"], cfg["y"], cfg["C"]) if cfg["task"] == "csvc" else \
    P.build_svr_dual(cfg["A"], cfg["t"], cfg["C"], cfg["epsilon"])
ts = []
for i in range(reps + 2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(torch.cuda.current_stream())
    r = P.alm_solve(pb, P.AlmOptions(tol_kkt=1e-6), return_device=True)
    e1.record(torch.cuda.current_stream())
    torch.cuda.synchronize()
    if i >= 2:
        ts.append(e0.elapsed_time(e1))
print(f"config {k}: median {statistics.median(ts):.3f} ms min {min(ts):.3f} ms  "
      f"outer {r.outer_iters} inner {r.total_inner_iters} kkt {r.kkt_residual:.2e}")
