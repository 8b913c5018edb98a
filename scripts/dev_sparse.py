import sys; sys.path.insert(0, '.')
import numpy as np, scipy.sparse as sp
import __graft_entry__ as g; g.build()
import paper_1910_01312_b200 as P
n, q, density, C = 3000, 400, 0.03, 1.0
rng = np.random.default_rng(n)
A = sp.random(n, q, density=density, random_state=rng, data_rvs=rng.standard_normal, format="csr")
w = np.zeros(q); w[rng.choice(q, size=8, replace=False)] = rng.standard_normal(8)
y = np.where(A @ w + 0.05 * rng.standard_normal(n) >= 0, 1.0, -1.0)
for name, feats, opts in (("dense", A.toarray(), P.SsnOptions()), ("csr", A, P.SsnOptions()), ("csr-cg2000", A, P.SsnOptions(cg_max_iters=5000))):
    rows = []
    pb = P.build_csvc_dual(feats, y, C)
    r = P.alm_solve(pb, P.AlmOptions(tol_kkt=1e-6), opts, callback=lambda *a: rows.append(a))
    print(name, r.converged, r.kkt_residual, r.outer_iters, r.total_inner_iters, r.objective, pb.native_counters)
    for row in rows: print('   ', row)
