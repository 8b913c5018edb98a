"""Dev: config-1-shaped X d and X^T v launches (L2 flushed) for ncu."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch
import __graft_entry__ as g; g.build()
from paper_1910_01312_b200.backend import default_backend
from paper_1910_01312_b200 import operators
be = default_backend()
rng = np.random.default_rng(0)
n, q = int(sys.argv[1]), int(sys.argv[2])
A = torch.from_numpy(rng.standard_normal((n, q))).cuda()
y = torch.from_numpy(np.where(rng.random(n) < .5, 1., -1.)).cuda()
op = operators.LinearKernelOperator(A, labels=y)
v = torch.from_numpy(rng.standard_normal(n)).cuda(); d = torch.from_numpy(rng.standard_normal((1, q))).cuda()
gr = be.empty((2, q)); out = be.empty((1, n))
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
for _ in range(2):
    flush.fill_(1); op.x(d, out, k=1)
    flush.fill_(1); op.xt([v], gr)
torch.cuda.synchronize()
