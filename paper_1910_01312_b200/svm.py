"""C-SVC and eps-SVR dual builders (linear kernel) and bias recovery.

Mirrors ref svm.py:95-127 (build_csvc_dual / build_svr_dual) and :147-208
(recover_bias).  The Q operator is the device-resident factor form of
operators.LinearKernelOperator; nothing n x n is formed.
"""

import numpy as np
import torch

from .backend import as_device, default_backend
from .errors import InputError
from .operators import LinearKernelOperator
from .projection import BoxLineSet
from .solver import QpProblem

SUPPORT_TOL = 1e-6  # ref svm.py:39


def _is_sparse(features):
    """scipy sparse matrix or an (indptr, indices, data, shape) CSR tuple."""
    if isinstance(features, tuple) and len(features) == 4:
        return True
    try:
        import scipy.sparse as sp

        return sp.issparse(features)
    except ImportError:  # pragma: no cover
        return False


def build_csvc_dual(features, labels, C, backend=None):
    """Q_ij = y_i y_j x_i'x_j, c = -e, y'x = 0, 0 <= x <= C (ref svm.py:95-108)."""
    be = backend or default_backend()
    y = np.asarray(labels.detach().cpu().numpy() if isinstance(labels, torch.Tensor) else labels,
                   dtype=np.float64)
    n = y.shape[0]
    if not np.all(np.abs(y) == 1.0):
        raise InputError("classification labels must be +1/-1")
    if n < 2 or np.unique(y).size < 2:
        raise InputError("need samples from both classes")
    if not C > 0:
        raise InputError("C must be positive")
    if _is_sparse(features):
        from .operators import CsrKernelOperator

        op = CsrKernelOperator(features, labels=y, backend=be)
    else:
        op = LinearKernelOperator(features, labels=y, backend=be)
    if op.n != n:
        raise InputError("labels must have one entry per sample")
    box = BoxLineSet(a=y, d=0.0, l=np.zeros(n), u=np.full(n, float(C)), backend=be,
                     a_device=op.row_sign)
    return QpProblem(op, torch.full((n,), -1.0, dtype=torch.float64, device=be.device), box)


def build_svr_dual(features, targets, C, epsilon, backend=None):
    """2n-variable regression dual: X = [A; -A], c = (eps - t; eps + t),
    a = (e; -e), d = 0, bounds [0, C] (ref svm.py:111-127)."""
    be = backend or default_backend()
    t = np.asarray(targets.detach().cpu().numpy() if isinstance(targets, torch.Tensor)
                   else targets, dtype=np.float64)
    n = t.shape[0]
    if not C > 0 or epsilon < 0:
        raise InputError("need C > 0 and epsilon >= 0")
    op = LinearKernelOperator(features, svr_block=True, backend=be)
    if op.n_phys != n:
        raise InputError("targets must have one entry per sample")
    # c = (eps - t; eps + t) and a = (e; -e) formed on the device from ONE upload of t
    t_dev = as_device(t, be)
    c = torch.cat([epsilon - t_dev, epsilon + t_dev])
    a_dev = torch.cat([torch.ones(n, dtype=torch.float64, device=be.device),
                       torch.full((n,), -1.0, dtype=torch.float64, device=be.device)])
    a = np.concatenate([np.ones(n), -np.ones(n)])
    box = BoxLineSet(a=a, d=0.0, l=np.zeros(2 * n), u=np.full(2 * n, float(C)), backend=be,
                     a_device=a_dev)
    return QpProblem(op, c, box)


def primal_weights(problem, dual_x):
    """w = X^T x (the linear model's weight vector, device tensor of length q)."""
    op = problem.q_op
    x = as_device(dual_x, op.backend)
    return op.xt([x])[0]


def recover_bias(problem, dual_x, targets, C, task="classification", epsilon=0.0):
    """Bias from the KKT conditions over free duals (ref svm.py:147-208)."""
    op = problem.q_op
    x = np.asarray(dual_x.detach().cpu().numpy() if isinstance(dual_x, torch.Tensor) else dual_x)
    w = primal_weights(problem, x)
    g = op.x(w.view(1, -1))[0][: op.n_phys].cpu().numpy()  # decision values (sign-free part)
    if op.row_sign is not None:
        g = g * op.row_sign.cpu().numpy()
    tol = SUPPORT_TOL * C
    t = np.asarray(targets, dtype=np.float64)
    if task == "classification":
        free = np.flatnonzero((x > tol) & (x < C - tol))
        if free.size:
            return float(np.mean(t[free] - g[free]))
        lows, highs = [], []
        for i in range(x.size):
            at_lower = x[i] <= tol
            if t[i] > 0:
                (lows if at_lower else highs).append(1.0 - g[i])
            else:
                (highs if at_lower else lows).append(-1.0 - g[i])
        return _interval_midpoint(lows, highs)
    n = op.n_phys
    xp, zp = x[:n], x[n:]
    contribs = list(t[(xp > tol) & (xp < C - tol)] - epsilon - g[(xp > tol) & (xp < C - tol)])
    contribs += list(t[(zp > tol) & (zp < C - tol)] + epsilon - g[(zp > tol) & (zp < C - tol)])
    if contribs:
        return float(np.mean(contribs))
    lows, highs = [], []
    for i in range(n):
        (lows if xp[i] <= tol else highs).append(t[i] - epsilon - g[i])
        (highs if zp[i] <= tol else lows).append(t[i] + epsilon - g[i])
    return _interval_midpoint(lows, highs)


def _interval_midpoint(lows, highs):
    if lows and highs:
        return float((max(lows) + min(highs)) / 2.0)
    if lows:
        return float(max(lows))
    if highs:
        return float(min(highs))
    return 0.0
