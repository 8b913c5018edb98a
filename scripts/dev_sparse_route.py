"""Dev: same sparse C-SVC through the direct and CG routes, debug lines on stderr."""
import sys; sys.path.insert(0, '.')
import numpy as np, scipy.sparse as sp
import __graft_entry__ as g; g.build()
import paper_1910_01312_b200 as P
n, q, density, C = 3000, 400, 0.03, 1.0
rng = np.random.default_rng(n)
A = sp.random(n, q, density=density, random_state=rng, data_rvs=rng.standard_normal, format="csr")
w = np.zeros(q); w[rng.choice(q, size=8, replace=False)] = rng.standard_normal(8)
y = np.where(A @ w + 0.05 * rng.standard_normal(n) >= 0, 1.0, -1.0)
thr = int(sys.argv[1])
rows = []
r = P.alm_solve(P.build_csvc_dual(A, y, C), P.AlmOptions(tol_kkt=1e-6), P.SsnOptions(direct_solve_threshold=thr), callback=lambda *a: rows.append(a))
print('RESULT', thr, r.converged, r.kkt_residual, r.outer_iters, r.total_inner_iters, file=sys.stderr)
for row in rows: print('   ', row, file=sys.stderr)
