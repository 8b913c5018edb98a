"""Dev microbenchmarks of latency-bound kernels (CUDA events, warm, per call)."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch
import __graft_entry__ as g; g.build()
from paper_1910_01312_b200.backend import default_backend
from paper_1910_01312_b200 import projection
be = default_backend()
def timeit(fn, reps=50):
    """GPU time per call: the calls captured into one CUDA graph, replayed (no host gaps)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3): fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(reps): fn()
    gr.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gr.replay()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps
rng = np.random.default_rng(0)
for m in (32, 64, 115, 160, 200, 300, 500, 1000, 2000):
    B = rng.standard_normal((m, m + 5)); M0 = torch.from_numpy(np.eye(m) + 10 * B @ B.T / m).cuda()
    M = M0.clone(); b = torch.from_numpy(rng.standard_normal(m)).cuda(); x = be.empty(m); info = be.zeros(1, torch.int32)
    def f():
        M.copy_(M0); be.chol_solve(M, m, b, 1.0, x, info)
    t = timeit(f)
    tc = timeit(lambda: M.copy_(M0))
    xs = np.linalg.solve(M0.cpu().numpy(), b.cpu().numpy())
    print(f"chol m={m}: {t - tc:.1f} us  err={np.abs(x.cpu().numpy()-xs).max():.2e}")
for n in (50_000, 1_000_000):
    a = np.where(rng.random(n) < .5, 1., -1.); v = torch.from_numpy(rng.standard_normal(n)).cuda()
    box = projection.BoxLineSet(a, 0.0, np.zeros(n), np.ones(n))
    st = be.new_states(4); xo = be.empty((4, n)); fo = be.zeros((4, n), torch.uint8)
    Bv = torch.from_numpy(rng.standard_normal(n) * 1e-3).cuda()
    be.project(v, box, st, 1, x_out=xo, free_out=fo)
    lam = float(be.read_states(st.cpu())[0]['lam'])
    t1 = timeit(lambda: be.project(v, box, st, 1, x_out=xo, free_out=fo, hint=lam))
    t4 = timeit(lambda: be.project(v, box, st, 4, B=Bv, coefs=[1, .5, .25, .125], x_out=xo, free_out=fo, hint=lam))
    st8 = be.new_states(8); xo8 = be.empty((8, n)); fo8 = be.zeros((8, n), torch.uint8)
    t8 = timeit(lambda: be.project(v, box, st8, 8, B=Bv, coefs=[2.0 ** -k for k in range(8)], x_out=xo8, free_out=fo8, hint=lam))
    tc = timeit(lambda: be.project(v, box, st, 1, x_out=xo, free_out=fo, hint=0.0))
    print(f"project n={n}: warm T=1 {t1:.1f} us, warm T=4 {t4:.1f} us, T=8 {t8:.1f} us, cold-hint T=1 {tc:.1f} us, passes={be.read_states(st.cpu())[0]['passes']}")
    out = be.zeros(8)
    w = [torch.from_numpy(rng.standard_normal(n)).cuda() for _ in range(8)]
    for k in (1, 4):
        print(f"dots n={n} k={k}: {timeit(lambda: be.dots([(w[j], w[j+4]) for j in range(k)], out)):.1f} us")
    print(f"vec n={n}: {timeit(lambda: be.vec(2, 0.5, w[0], w[1], None, w[2])):.1f} us")
# streaming products on config-1 shapes (A 50000 x 300, 120 MB)
from paper_1910_01312_b200 import operators
n, q = 50_000, 300
A = torch.from_numpy(rng.standard_normal((n, q))).cuda()
y = torch.from_numpy(np.where(rng.random(n) < .5, 1., -1.)).cuda()
op = operators.LinearKernelOperator(A, labels=y)
v = torch.from_numpy(rng.standard_normal(n)).cuda(); d = torch.from_numpy(rng.standard_normal((1, q))).cuda()
gr = be.empty((2, q)); out = be.empty((1, n))
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
t_f = timeit(lambda: flush.fill_(1), reps=10)
t_xd = timeit(lambda: (flush.fill_(1), op.x(d, out, k=1)), reps=10) - t_f
t_xt = timeit(lambda: (flush.fill_(1), op.xt([v], gr)), reps=10) - t_f
t_xd_w = timeit(lambda: op.x(d, out, k=1), reps=20)
t_xt_w = timeit(lambda: op.xt([v], gr), reps=20)
gb = n * q * 8 / 1e9
print(f"xd cold {t_xd:.1f} us ({gb/t_xd*1e6:.0f} GB/s)  warm {t_xd_w:.1f} us ({gb/t_xd_w*1e6:.0f} GB/s)")
print(f"xt cold {t_xt:.1f} us ({gb/t_xt*1e6:.0f} GB/s)  warm {t_xt_w:.1f} us ({gb/t_xt_w*1e6:.0f} GB/s)")
dd = d[0].clone()
t_mv = timeit(lambda: (flush.fill_(1), torch.mv(A, dd)), reps=10) - t_f
t_sum = timeit(lambda: (flush.fill_(1), A.sum()), reps=10) - t_f
t_cp = timeit(lambda: (flush.fill_(1), flush[:n*q*8//2].copy_(flush[n*q*8//2:n*q*8])), reps=10) - t_f
print(f"reference points (cold): cuBLAS dgemv {t_mv:.1f} us ({gb/t_mv*1e6:.0f} GB/s), torch sum {t_sum:.1f} us ({gb/t_sum*1e6:.0f} GB/s), 60MB->60MB copy {t_cp:.1f} us ({gb/t_cp*1e6:.0f} GB/s r+w)")
