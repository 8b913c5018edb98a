"""Offline study (CPU, oracle): sample-space CG with a hot-column Woodbury preconditioner
on a 1/10-scale config-3 Newton system (n=400k, q=100k, Zipf).
  system   (I_p + sigma P K P) y = P g_J,  K = X_J X_J^T,  P = I - a a^T / a^T a
  precond  B = I + sigma X_H X_H^T  (H = the h hottest columns of X_J),
           B^-1 = I - X_H (I_h / sigma + X_H^T X_H)^-1 X_H^T
Stopping rule: the product's true Newton residual, checked every 16 iterations.
Usage: python scripts/precond_study2.py K [scale]   (captures at sigma = 5^K)"""
import sys
import time

import numpy as np
import scipy.linalg
import scipy.sparse as sp

sys.path.insert(0, ".")
import oracle as O
from oracle import ssnal_oracle as SO
from paper_1910_01312_b200 import datagen

K = int(sys.argv[1]) if len(sys.argv) > 1 else 4
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
cfg = datagen.config3(n=int(4_000_000 * scale), q=int(1_000_000 * scale))
op, c, bl = O.csvc_problem_csr(cfg["indptr"], cfg["indices"], cfg["data"], cfg["shape"], cfg["y"],
                               cfg["C"])
O.set_psi_mode("delta")
captured = {}
orig = SO.newton_direction_factor


class Stop(Exception):
    pass


def hook(s, grad, free, sigma, op_, a, opts):
    if sigma >= 5.0 ** K:
        captured.update(s=s.copy(), grad=grad.copy(), free=free.copy(), sigma=sigma)
        raise Stop
    return orig(s, grad, free, sigma, op_, a, opts)


SO.newton_direction_factor = hook
t0 = time.time()
try:
    O.alm_solve(op, c, bl, O.AlmOpts(tol_kkt=1e-6), O.SsnOpts(newton="factor", max_inner=200))
except Stop:
    pass
print(f"captured sigma={captured['sigma']} after {time.time() - t0:.0f}s", flush=True)
s, grad, free, sigma = captured["s"], captured["grad"], captured["free"], captured["sigma"]
J = np.flatnonzero(free)
p = J.size
xj = op.rows(J).tocsr()
xjT = xj.T.tocsr()
a_j = bl.a[J]
asa = float(a_j @ a_j)
g_j = grad[J]
q = xj.shape[1]
colsq = np.asarray(xj.multiply(xj).sum(axis=0)).ravel()
print(f"p={p} q={q} nnz(X_J)={xj.nnz} sigma={sigma}", flush=True)
gnorm = np.linalg.norm(grad)
target = min(1e-2, gnorm ** 1.5)
r_q = op.xt(s)


def proj(v):
    return v - (a_j @ v / asa) * a_j


def apply_k(y):  # (I + sigma P K P) y
    return y + sigma * proj(xj @ (xjT @ proj(y)))


def newton_res(y):
    # t = -r + sigma X_J^T P y; residual of the q-space system mapped to n-space
    t = -r_q + sigma * (xjT @ proj(y))
    z = xj @ t
    res_t = -r_q - (t + sigma * (xjT @ proj(z)))
    zz = xj @ res_t
    return np.linalg.norm(op.x(sigma * (xjT @ proj(zz))))


def pcg(apply_pre, name, cost, max_it=6000):
    b = proj(g_j)
    y = np.zeros(p)
    res = b.copy()
    z = apply_pre(res)
    pv = z.copy()
    rz = res @ z
    t0 = time.time()
    for it in range(1, max_it + 1):
        mp = apply_k(pv)
        al = rz / (pv @ mp)
        y += al * pv
        res -= al * mp
        if it % 16 == 0 and newton_res(y) <= target:
            break
        z = apply_pre(res)
        rz2 = res @ z
        pv = z + (rz2 / rz) * pv
        rz = rz2
    print(f"{name:22s} iterations {it:6d}  x cost {cost:.2f} = {it * cost:8.0f}  newton residual "
          f"{newton_res(y):.3e} (target {target:.3e})  {time.time() - t0:.1f}s", flush=True)


pcg(lambda v: v, "pspace none", 1.0)
order = np.argsort(-colsq)
for h in [int(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else "64,256,1024,4096".split(","))]:
    H = np.sort(order[:h])
    xh = xj[:, H].tocsr()
    xhT = xh.T.tocsr()
    frac = xh.nnz / xj.nnz
    # the preconditioner must commute with range(P): use P B P restricted -> include a in the low-rank part
    U = sp.hstack([xh, sp.csr_matrix(a_j.reshape(-1, 1) / np.sqrt(asa))]).tocsr()
    GH = (xhT @ xh).toarray()
    M = np.eye(h) / sigma + GH
    cf = scipy.linalg.cho_factor(M, lower=True)

    def pre(v, xh=xh, xhT=xhT, cf=cf):
        w = proj(v)
        w = w - xh @ scipy.linalg.cho_solve(cf, xhT @ w)
        return proj(w)

    pcg(pre, f"pspace hot-{h}", 1.0 + frac)
    print(f"   hot fraction of nnz: {frac:.3f}; next column norm^2 {colsq[order[h]]:.2f}", flush=True)
