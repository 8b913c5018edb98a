"""Where the config-4 end-to-end time goes: pinned H2D of A, problem construction, solve,
read-back (CUDA events + host clocks)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import __graft_entry__ as g

g.build()
import paper_1910_01312_b200 as P
from paper_1910_01312_b200 import datagen

cfg = datagen.make_config(4)
A_host = torch.from_numpy(cfg["A"]).pin_memory()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Ad = A_host.to("cuda", non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    pb = P.build_svr_dual(Ad, cfg["t"], cfg["C"], cfg["epsilon"])
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    r = P.alm_solve(pb, P.AlmOptions(tol_kkt=1e-6))
    t3 = time.perf_counter()
    print(f"H2D {t1 - t0:.4f} s ({A_host.numel() * 8 / (t1 - t0) / 1e9:.1f} GB/s), build {t2 - t1:.4f} s, "
          f"solve+readback {t3 - t2:.4f} s", flush=True)
    del Ad, pb
