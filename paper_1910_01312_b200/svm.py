"""C-SVC and eps-SVR pipelines on the device solver (linear kernel).

Mirrors ref svm.py: SvmConfig (:42-63), SvmModel (:66-77), build_csvc_dual /
build_svr_dual (:95-127), recover_bias (:147-208, with _support_from_dual :136-144 and
_interval_midpoint :211-218), decision_function / predict / evaluate (:221-245),
train (:269-295) -- same names, argument meaning and errors.  The Q operator is the
device-resident factor form (operators.LinearKernelOperator / CsrKernelOperator);
nothing n x n is formed.  Decision values for the bias come from two device products
(w = A^T coef, g = A w) and the free-set means / interval bounds from device reductions.

Out of scope: RBF kernels and the Nystrom / RFF approximations,
cross-validation, model files.  A config asking for them raises InputError.
"""

from dataclasses import dataclass, field

import numpy as np
import torch

from .backend import as_device, default_backend
from .errors import InputError
from .operators import LinearKernelOperator
from .projection import BoxLineSet
from .solver import QpProblem

CLASSIFICATION = "classification"
REGRESSION = "regression"
APPROX_EXACT = "exact"
LINEAR = "linear"
SUPPORT_TOL = 1e-6  # ref svm.py:39


@dataclass(frozen=True)
class KernelSpec:
    """Kernel family and width (ref kernels.py:27-39); the device path is linear."""

    kind: str = LINEAR
    alpha: float = 1.0

    def __post_init__(self):
        if self.kind not in (LINEAR, "rbf"):
            raise InputError(f"unknown kernel kind {self.kind!r}")
        if self.kind == "rbf" and not self.alpha > 0:
            raise InputError("RBF width alpha must be positive")


@dataclass(frozen=True)
class SvmConfig:
    """ref svm.py:42-63 (same fields and validation)."""

    task: str = CLASSIFICATION
    C: float = 1.0
    kernel: KernelSpec = field(default_factory=KernelSpec)
    epsilon: float = 0.0
    approx: str = APPROX_EXACT
    approx_size: int = 0
    seed: int = 0

    def __post_init__(self):
        if self.task not in (CLASSIFICATION, REGRESSION):
            raise InputError(f"unknown task {self.task!r}")
        if not self.C > 0:
            raise InputError("C must be positive")
        if self.epsilon < 0:
            raise InputError("epsilon must be non-negative")
        if self.approx not in (APPROX_EXACT, "nystrom", "rff"):
            raise InputError(f"unknown approximation {self.approx!r}")
        if self.approx != APPROX_EXACT and self.approx_size < 1:
            raise InputError("approximation size must be at least 1")


def _check_linear_exact(config):
    if config.kernel.kind != LINEAR or config.approx != APPROX_EXACT:
        raise InputError("the device path solves the linear-kernel dual exactly; RBF kernels "
                         "and Nystrom/RFF approximations are out of scope (DESIGN.md section 10)")


@dataclass
class SvmModel:
    """Trained model (ref svm.py:66-77)."""

    config: SvmConfig
    bias: float
    dual_x: np.ndarray
    support_indices: np.ndarray
    support_coef: np.ndarray
    support_features: np.ndarray
    n_train: int
    q: int


def _is_sparse(features):
    """scipy sparse matrix or an (indptr, indices, data, shape) CSR tuple."""
    if isinstance(features, tuple) and len(features) == 4:
        return True
    try:
        import scipy.sparse as sp

        return sp.issparse(features)
    except ImportError:  # pragma: no cover
        return False


def _config_and_c(config_or_c, epsilon=None, task=CLASSIFICATION):
    """Accept the reference's SvmConfig or (back-compatible) a bare C [, epsilon]."""
    if isinstance(config_or_c, SvmConfig):
        _check_linear_exact(config_or_c)
        return config_or_c
    C = float(config_or_c)
    if not C > 0:
        raise InputError("C must be positive")
    eps = 0.0 if epsilon is None else float(epsilon)
    if eps < 0:
        raise InputError("epsilon must be non-negative")
    return SvmConfig(task=task, C=C, epsilon=eps)


def _host_vector(v):
    return np.asarray(v.detach().cpu().numpy() if isinstance(v, torch.Tensor) else v,
                      dtype=np.float64)


def build_csvc_dual(features, labels, config, backend=None):
    """Classification dual: Q_ij = y_i y_j x_i'x_j, c = -e, y'x = 0, 0 <= x <= C
    (ref svm.py:95-108).  ``config``: SvmConfig (or C)."""
    cfg = _config_and_c(config)
    be = backend or default_backend()
    y = _host_vector(labels)
    n = y.shape[0]
    if y.ndim != 1:
        raise InputError("labels must have one entry per sample")
    pos = y == 1.0
    if not np.all(pos | (y == -1.0)):
        raise InputError("classification labels must be +1/-1")
    if n < 2 or pos.all() or not pos.any():  # (np.unique sorts: 0.3 s at n = 4M)
        raise InputError("need samples from both classes")
    if _is_sparse(features):
        from .operators import CsrKernelOperator

        op = CsrKernelOperator(features, labels=y, backend=be)
    else:
        op = LinearKernelOperator(features, labels=y, backend=be)
    if op.n != n:
        raise InputError("labels must have one entry per sample")
    box = BoxLineSet(a=y, d=0.0, l=0.0, u=cfg.C, backend=be, a_device=op.row_sign)
    return QpProblem(op, torch.full((n,), -1.0, dtype=torch.float64, device=be.device), box)


def build_svr_dual(features, targets, config, epsilon=None, backend=None):
    """Regression dual over 2n variables (x, z): X = [A; -A], c = (eps - t; eps + t),
    a = (e; -e), d = 0, bounds [0, C] (ref svm.py:111-127).  ``config``: SvmConfig (or C,
    with ``epsilon``)."""
    cfg = _config_and_c(config, epsilon, REGRESSION)
    be = backend or default_backend()
    t = _host_vector(targets)
    n = t.shape[0]
    if t.ndim != 1:
        raise InputError("targets must have one entry per sample")
    op = LinearKernelOperator(features, svr_block=True, backend=be)
    if op.n_phys != n:
        raise InputError("targets must have one entry per sample")
    # c = (eps - t; eps + t) and a = (e; -e) formed on the device from ONE upload of t
    eps = cfg.epsilon
    t_dev = as_device(t, be)
    c = torch.cat([eps - t_dev, eps + t_dev])
    a_dev = torch.cat([torch.ones(n, dtype=torch.float64, device=be.device),
                       torch.full((n,), -1.0, dtype=torch.float64, device=be.device)])
    a = np.concatenate([np.ones(n), -np.ones(n)])
    box = BoxLineSet(a=a, d=0.0, l=0.0, u=cfg.C, backend=be, a_device=a_dev)
    return QpProblem(op, c, box)


def primal_weights(problem, dual_x):
    """w = X^T x (the linear model's weight vector, device tensor of length q)."""
    op = problem.q_op
    x = as_device(dual_x, op.backend)
    return op.xt([x])[0]


def _unsigned_operator(features, problem, be):
    """The sample matrix A as a label-free device operator (the reference's decision
    values use K(x_j, .) without labels).  Reuses the problem's device copy of A."""
    op = getattr(problem, "q_op", None) if problem is not None else None
    if op is not None and getattr(op, "kind", "") == "dense":
        return LinearKernelOperator(op.A, backend=be)
    if op is not None and getattr(op, "kind", "") == "csr" and op.row_sign is None:
        return op
    if _is_sparse(features):
        from .operators import CsrKernelOperator

        return CsrKernelOperator(features, backend=be)
    return LinearKernelOperator(features, backend=be)


def _support_coef(x, config, n_phys):
    """ref svm.py:136-144: coefficients with |coef| > SUPPORT_TOL * C kept."""
    tol = SUPPORT_TOL * config.C
    coef = x if config.task == CLASSIFICATION else x[:n_phys] - x[n_phys:]
    keep = coef.abs() > tol
    return torch.where(keep, coef, torch.zeros_like(coef)), keep


def _interval_midpoint(lo_vals, hi_vals):
    """ref svm.py:211-218 on device vectors (max of lows, min of highs)."""
    have_lo, have_hi = lo_vals.numel() > 0, hi_vals.numel() > 0
    if have_lo and have_hi:
        return float((lo_vals.max() + hi_vals.min()) / 2.0)
    if have_lo:
        return float(lo_vals.max())
    if have_hi:
        return float(hi_vals.min())
    return 0.0


def recover_bias(dual_x, features, targets, config, problem=None, backend=None):
    """Bias from the KKT conditions of the solved dual (ref svm.py:147-208).

    Averages the KKT equation over free duals (strictly between the bounds); with no
    free dual, the midpoint of the interval the bound-active conditions leave feasible.
    Decision values g = A (A_sv^T coef_sv) use the support vectors only, without labels,
    as the reference's kernel path does.  ``problem`` (optional) lends its device copy of
    A; otherwise ``features`` is uploaded."""
    cfg = _config_and_c(config)
    be = backend or (problem.backend if problem is not None else default_backend())
    x = as_device(dual_x, be).reshape(-1)
    if x.numel() == 0:
        raise InputError("empty dual solution")
    t = as_device(targets, be).reshape(-1)
    cc = cfg.C
    tol = SUPPORT_TOL * cc
    A = _unsigned_operator(features, problem, be)
    n = A.n_phys
    coef, _ = _support_coef(x, cfg, n)
    w = A.xt([coef])[0]                     # A^T coef (device product)
    g = A.x(w.view(1, -1))[0][:n]           # decision values (device product)
    if cfg.task == CLASSIFICATION:
        free = (x > tol) & (x < cc - tol)
        if bool(free.any()):
            return float((t[free] - g[free]).mean())
        at_lower = x <= tol
        pos = t > 0
        lows = torch.cat([(1.0 - g)[pos & at_lower], (-1.0 - g)[~pos & ~at_lower]])
        highs = torch.cat([(1.0 - g)[pos & ~at_lower], (-1.0 - g)[~pos & at_lower]])
        return _interval_midpoint(lows, highs)
    eps = cfg.epsilon
    xp, zp = x[:n], x[n:]
    fx = (xp > tol) & (xp < cc - tol)
    fz = (zp > tol) & (zp < cc - tol)
    contribs = torch.cat([(t - eps - g)[fx], (t + eps - g)[fz]])
    if contribs.numel():
        return float(contribs.mean())
    lx, lz = xp <= tol, zp <= tol
    lows = torch.cat([(t - eps - g)[lx], (t + eps - g)[~lz]])
    highs = torch.cat([(t - eps - g)[~lx], (t + eps - g)[lz]])
    return _interval_midpoint(lows, highs)


def _host_rows(features, idx):
    if _is_sparse(features):
        import scipy.sparse as sp

        if isinstance(features, tuple):
            indptr, indices, data, shape = features
            features = sp.csr_matrix((data, indices, indptr), shape=shape)
        return features[idx]
    f = features.detach().cpu().numpy() if isinstance(features, torch.Tensor) else features
    return np.asarray(f, dtype=np.float64)[idx].copy()


def _make_model(dual_x, features, targets, config, problem=None):
    """ref svm.py:238-250."""
    x = as_device(dual_x, problem.backend if problem is not None else default_backend())
    n = x.numel() if config.task == CLASSIFICATION else x.numel() // 2
    coef, keep = _support_coef(x, config, n)
    sv_idx = torch.nonzero(keep, as_tuple=False).flatten().cpu().numpy()
    bias = recover_bias(x, features, targets, config, problem=problem)
    q = problem.q_op.q if problem is not None else np.asarray(features).shape[1]
    return SvmModel(config=config, bias=bias, dual_x=x.cpu().numpy(), support_indices=sv_idx,
                    support_coef=coef[keep].cpu().numpy(),
                    support_features=_host_rows(features, sv_idx), n_train=n, q=int(q))


def train(features, targets, config, alm_opts=None, ssn_opts=None, warm_start_freqs=None):
    """Build the dual, solve it on the device, package the model (ref svm.py:269-295).
    Returns ``(model, report)``."""
    from .solver import alm_solve

    _check_linear_exact(config)
    if warm_start_freqs:
        raise InputError("the RFF warm start is out of scope (DESIGN.md section 10)")
    if config.task == CLASSIFICATION:
        problem = build_csvc_dual(features, targets, config)
    else:
        problem = build_svr_dual(features, targets, config)
    report = alm_solve(problem, alm_opts=alm_opts, ssn_opts=ssn_opts)
    model = _make_model(report.x_opt, features, targets, config, problem=problem)
    return model, report


def decision_function(model, points):
    """Decision values / regression estimates (ref svm.py:221-229): points @ w + b with
    w = support_features^T support_coef, both products on the device."""
    pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
    if pts.shape[1] != model.q:
        raise InputError(f"expected {model.q} features, got {pts.shape[1]}")
    be = default_backend()
    if model.support_coef.size == 0:
        return np.full(pts.shape[0], model.bias)
    sv = model.support_features
    sv = sv.toarray() if hasattr(sv, "toarray") else sv
    w = LinearKernelOperator(sv, backend=be).xt([as_device(model.support_coef, be)])[0]
    g = LinearKernelOperator(pts, backend=be).x(w.view(1, -1))[0]
    return g.cpu().numpy() + model.bias


def predict(model, point):
    """ref svm.py:232-234."""
    return float(decision_function(model, np.asarray(point, dtype=float)[None, :])[0])


def evaluate(model, features, targets):
    """Accuracy (classification) or mean squared error (regression); ref svm.py:237-245."""
    targets = np.asarray(targets, dtype=float)
    if targets.size == 0:
        raise InputError("empty test set")
    values = decision_function(model, features)
    if model.config.task == CLASSIFICATION:
        pred = np.where(values >= 0.0, 1.0, -1.0)
        return {"accuracy": float(np.mean(pred == targets))}
    return {"mse": float(np.mean((targets - values) ** 2))}
