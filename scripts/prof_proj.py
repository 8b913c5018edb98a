"""Dev: warm-started projections (T=1 and T=4) for ncu."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch
import __graft_entry__ as g; g.build()
from paper_1910_01312_b200.backend import default_backend
from paper_1910_01312_b200 import projection
be = default_backend()
rng = np.random.default_rng(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
a = np.where(rng.random(n) < .5, 1., -1.); v = torch.from_numpy(rng.standard_normal(n)).cuda()
box = projection.BoxLineSet(a, 0.0, np.zeros(n), np.ones(n))
st = be.new_states(4); xo = be.empty((4, n)); fo = be.zeros((4, n), torch.uint8)
Bv = torch.from_numpy(rng.standard_normal(n) * 1e-3).cuda()
be.project(v, box, st, 1, x_out=xo, free_out=fo)
lam = float(be.read_states(st.cpu())[0]['lam'])
for _ in range(3):
    be.project(v, box, st, 1, x_out=xo, free_out=fo, hint=lam)
    be.project(v, box, st, 4, B=Bv, coefs=[1, .5, .25, .125], x_out=xo, free_out=fo, hint=lam)
torch.cuda.synchronize()
