"""Dev: one chol_solve launch per size for ncu."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch
import __graft_entry__ as g; g.build()
from paper_1910_01312_b200.backend import default_backend
be = default_backend()
rng = np.random.default_rng(0)
for m in [int(a) for a in sys.argv[1:]]:
    B = rng.standard_normal((m, m + 5)); M = torch.from_numpy(np.eye(m) + 10 * B @ B.T / m).cuda()
    b = torch.from_numpy(rng.standard_normal(m)).cuda(); x = be.empty(m); info = be.zeros(1, torch.int32)
    be.chol_solve(M, m, b, 1.0, x, info)
torch.cuda.synchronize()
