"""Offline study (CPU, oracle): CG iterations of the config-3 Newton system under
different preconditioners, on a 1/10-scale config-3 problem (n=400k, q=100k, Zipf).
Captures the factor-space system (I + sigma X_J^T P X_J) t = -X^T s at the first Newton
step of outer iteration K, then runs PCG to the product's stopping rule with:
  jacobi          diag(1 + sigma max(colsq - m1^2/asa, 0))
  hot-block-k     exact (I + sigma G_HH - ...) on the k hottest columns + Jacobi elsewhere
  pspace          CG on the p x p dual (I + sigma P Q_JJ P) y = P g_J (no preconditioner)
"""
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
cfg = datagen.config3(n=400_000, q=100_000)
op, c, bl = O.csvc_problem_csr(cfg["indptr"], cfg["indices"], cfg["data"], cfg["shape"], cfg["y"],
                               cfg["C"])
O.set_psi_mode("delta")
captured = {}
orig = SO.newton_direction_factor
calls = {"outer": -1, "n": 0}


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
a_j = bl.a[J]
asa = float(a_j @ a_j)
r = op.xt(s)
m1 = np.asarray(xj.T @ a_j).ravel()
colsq = np.asarray(xj.multiply(xj).sum(axis=0)).ravel()
q = r.size
print(f"p={p} q={q} nnz(X_J)={xj.nnz} sigma={sigma}", flush=True)
xjT = xj.T.tocsr()


def gram_p(v):
    z = xj @ v
    z = z - (a_j @ z / asa) * a_j
    return xjT @ z


gnorm = np.linalg.norm(grad)
target = 0.1 * min(1e-2, 1e-4, gnorm ** 1.5)


def newton_res(t):
    res = -r - (t + sigma * gram_p(t))
    return np.linalg.norm(op.x(sigma * gram_p(res)))


def pcg(apply_pre, name, max_it=20000):
    v = np.zeros(q)
    res = -r.copy()
    z = apply_pre(res)
    pv = z.copy()
    rz = res @ z
    t0 = time.time()
    for it in range(1, max_it + 1):
        mp = pv + sigma * gram_p(pv)
        al = rz / (pv @ mp)
        v += al * pv
        res -= al * mp
        if it % 16 == 0 and newton_res(v) <= target:
            break
        z = apply_pre(res)
        rz2 = res @ z
        pv = z + (rz2 / rz) * pv
        rz = rz2
    print(f"{name:18s} iterations {it:6d}  newton residual {newton_res(v):.3e} (target {target:.3e})"
          f"  {time.time() - t0:.1f}s", flush=True)


dj = 1.0 + sigma * np.maximum(colsq - m1 * m1 / asa, 0.0)
pcg(lambda v: v / dj, "jacobi")
pcg(lambda v: v, "none (identity)")
order = np.argsort(-colsq)
for k in (64, 256, 1024):
    H = np.sort(order[:k])
    XH = xj[:, H].toarray()
    GH = XH.T @ XH - np.outer(m1[H], m1[H]) / asa
    MH = np.eye(k) + sigma * GH
    cf = scipy.linalg.cho_factor(MH, lower=True)
    rest = np.ones(q, bool)
    rest[H] = False

    def pre(v, H=H, cf=cf, rest=rest):
        out = np.empty_like(v)
        out[H] = scipy.linalg.cho_solve(cf, v[H])
        out[rest] = v[rest] / dj[rest]
        return out

    def pre_id(v, H=H, cf=cf, rest=rest):
        out = v.copy()
        out[H] = scipy.linalg.cho_solve(cf, v[H])
        return out

    pcg(pre, f"hot-block-{k}+jac")
    pcg(pre_id, f"hot-block-{k}+id")

