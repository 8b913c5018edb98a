import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
import __graft_entry__ as g; g.build()
import paper_1910_01312_b200 as P
from paper_1910_01312_b200 import datagen
cfg = datagen.config1()
A_host = torch.from_numpy(cfg["A"]).pin_memory(); y = cfg["y"]
for i in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pb = P.build_csvc_dual(A_host, y, cfg["C"]); torch.cuda.synchronize(); t1 = time.perf_counter()
    r = P.alm_solve(pb, P.AlmOptions(tol_kkt=1e-6)); torch.cuda.synchronize(); t2 = time.perf_counter()
    Ad = torch.empty_like(A_host, device='cuda'); torch.cuda.synchronize(); t3 = time.perf_counter()
    Ad.copy_(A_host, non_blocking=True); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"build {1e3*(t1-t0):.2f} ms  solve {1e3*(t2-t1):.2f} ms  (h2d alone {1e3*(t4-t3):.2f} ms, {A_host.numel()*8/(t4-t3)/1e9:.1f} GB/s)")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
pb = P.build_csvc_dual(A_host, y, cfg["C"]); torch.cuda.synchronize()
pr.disable(); pstats.Stats(pr).sort_stats('cumulative').print_stats(12)
