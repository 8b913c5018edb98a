import sys; sys.path.insert(0, '.')
import numpy as np, torch
import __graft_entry__ as g; g.build()
from paper_1910_01312_b200.backend import default_backend
be = default_backend()
def timeit(fn, reps=50):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3): fn()
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(reps): fn()
    gr.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); gr.replay(); e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps
rng = np.random.default_rng(0)
for m in (300, 500, 1000, 2000):
    B = rng.standard_normal((m, m + 5)); M0 = torch.from_numpy(np.eye(m) + 10 * B @ B.T / m).cuda()
    M = M0.clone(); b = torch.from_numpy(rng.standard_normal(m)).cuda(); x = be.empty(m); info = be.zeros(1, torch.int32)
    def f():
        M.copy_(M0); be.chol_solve(M, m, b, 1.0, x, info)
    t = timeit(f); tc = timeit(lambda: M.copy_(M0))
    print(f"chol m={m}: {t - tc:.1f} us")
