"""Time the large-n projection (multi-trial cooperative kernel) on eps-SVR-shaped data:
T trials of v_t = u - c_t Qd, warm hint near the root, CUDA events, passes per trial."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import __graft_entry__ as g

g.build()
import paper_1910_01312_b200 as P

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
n = 2 * m
rng = np.random.default_rng(0)
a = np.concatenate([np.ones(m), -np.ones(m)])
box = P.BoxLineSet(a, 0.0, np.zeros(n), np.ones(n))
be = box.backend
# u: most slots saturated far outside [0, 1], a few thousand near the box
u = rng.standard_normal(n) * 50.0
near = rng.choice(n, size=20000, replace=False)
u[near] = rng.random(near.size) * 1.2 - 0.1
qd = rng.standard_normal(n) * 0.01
ud = torch.as_tensor(u, device="cuda")
qdd = torch.as_tensor(qd, device="cuda")
for T in (1, 2, 4, 8):
    coefs = [1.0 * 0.5 ** j for j in range(T)]
    states = be.new_states(T)
    xo = be.empty((T, n))
    fo = be.empty((T, n), torch.uint8)
    st = be.project_sync(ud, box, states, T=T, B=qdd, coefs=coefs, x_out=xo, free_out=fo)
    lam = float(st["lam"][0])
    ts = []
    for rep in range(10):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        be.project(ud, box, states, T, qdd, coefs, xo, fo, hint=lam * (1 + 1e-4))
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    st = be.read_states(states[:T].cpu())
    print(f"T={T}: {np.median(ts):8.1f} us  passes={list(st['passes'])} status={list(st['status'])}")
