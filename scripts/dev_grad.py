import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
import __graft_entry__ as g; g.build()
import paper_1910_01312_b200 as P
from conftest import load_cases
be = P.default_backend()
for i, c in enumerate(load_cases("solve.npz", "s")):
    if c["kind"] == "dense":
        pb = P.QpProblem(P.DenseOperator(c["G"].T @ c["G"]), c["c"], P.BoxLineSet(c["a"], c["d"], c["l"], c["u"]))
    elif c["kind"] == "csvc":
        pb = P.build_csvc_dual(c["A"], c["y"], c["C"])
    else:
        pb = P.build_svr_dual(c["A"], c["t"], c["C"], c["eps"])
    op = pb.q_op; n, q = pb.n, op.q
    rng = np.random.default_rng(i)
    w = torch.from_numpy(rng.standard_normal(n)).cuda(); xp = torch.from_numpy(rng.standard_normal(n)).cuda()
    s = be.empty(n); gr = be.empty((2, q)); grad = be.empty(n); g2 = be.zeros(16)
    be.dense_gradient(op, w, xp, s, gr[0], grad, g2[4:5])
    s2 = w - xp; gr2 = op.xt([s2]); grad2 = op.x(gr2)[0]
    torch.cuda.synchronize()
    print(i, c["kind"], n, q, op.lda, op.A.data_ptr() % 16, float((s - s2).abs().max()), float((gr[0] - gr2[0]).abs().max()), float((grad - grad2).abs().max()), float(g2[4]), float(grad2 @ grad2))
