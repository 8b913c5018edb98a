"""Projection onto {x : a'x = d, l <= x <= u} and its HS-Jacobian (device API).

Mirrors ref projection.py (BoxLineSet :22-57, ActiveSetMask :60-79,
ProjectionResult :82-105, project_box_line :152-211, hs_jacobian_apply
:214-225): same names, argument meaning and errors.  Vectors may be numpy
arrays or torch tensors; results are CUDA tensors.  The arithmetic runs in
the sm_100a library (csrc/proj.cu, csrc/vec.cu).
"""

import numpy as np
import torch

from . import _lib
from .backend import as_device, check_vector, default_backend
from .errors import InfeasibleProblemError, InputError


def _uniform_value(t):
    """Python float if every entry of the device vector is equal, else None."""
    lo, hi = torch.aminmax(t)
    lo, hi = float(lo), float(hi)
    return lo if lo == hi else None


class BoxLineSet:
    """Constraint set {x : a'x = d, l <= x <= u}; feasibility checked once at
    construction (ref projection.py:29-54).  Constant bounds are passed to the
    kernels as scalars (no l/u streams)."""

    def __init__(self, a, d, l, u, backend=None, a_device=None):
        self.backend = backend or default_backend()
        a_h = np.ascontiguousarray(a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a,
                                   dtype=np.float64)
        if a_h.ndim != 1:
            raise InputError("a, l, u must be one-dimensional vectors of equal length")
        n = a_h.shape[0]
        d = float(d)
        # l / u: vectors as in the reference, or scalars (a constant bound for every slot:
        # the SVM builders pass l = 0, u = C and skip three passes over n-length arrays)
        l_uniform, l_c, l_h = self._bound(l, n)
        u_uniform, u_c, u_h = self._bound(u, n)
        if l_uniform and u_uniform:
            if not l_c < u_c:
                raise InputError("box must satisfy l < u componentwise")
            a_sum = float(a_h.sum())
            a_abs = float(np.abs(a_h).sum())
            pos, neg = 0.5 * (a_sum + a_abs), 0.5 * (a_sum - a_abs)  # sums of a_i > 0, a_i < 0
            lo, hi = pos * l_c + neg * u_c, pos * u_c + neg * l_c
        else:
            l_v = l_h if l_h is not None else np.full(n, l_c)
            u_v = u_h if u_h is not None else np.full(n, u_c)
            if not np.all(l_v < u_v):
                raise InputError("box must satisfy l < u componentwise")
            lo = float(np.sum(np.where(a_h > 0, a_h * l_v, a_h * u_v)))
            hi = float(np.sum(np.where(a_h > 0, a_h * u_v, a_h * l_v)))
        slack = 1e-12 * (1.0 + abs(d) + max(abs(lo), abs(hi)))
        if not (lo - slack <= d <= hi + slack):
            raise InfeasibleProblemError(
                f"a'x = {d} unattainable over the box: range is [{lo}, {hi}]")
        self.n = n
        self.d = d
        # a_device: the caller's device copy of the same values (e.g. the labels already
        # uploaded for the operator), saving a second upload
        self.a_dev = a_device if a_device is not None else as_device(a_h, self.backend)
        self.l_const = l_c if l_uniform else 0.0
        self.u_const = u_c if u_uniform else 0.0
        self.l_dev = None if l_uniform else as_device(l_h, self.backend)
        self.u_dev = None if u_uniform else as_device(u_h, self.backend)
        self._range_lo, self._range_hi = lo, hi

    @staticmethod
    def _bound(b, n):
        """(uniform, constant, host vector or None) for a scalar or an n-vector bound."""
        if np.isscalar(b) or (isinstance(b, np.ndarray) and b.ndim == 0):
            return True, float(b), None
        b_h = np.ascontiguousarray(b.detach().cpu().numpy() if isinstance(b, torch.Tensor) else b,
                                   dtype=np.float64)
        if b_h.shape != (n,):
            raise InputError("a, l, u must be one-dimensional vectors of equal length")
        if n and bool(np.all(b_h == b_h[0])):
            return True, float(b_h[0]), None
        return False, 0.0, b_h

    @property
    def a(self):
        return self.a_dev

    @property
    def l(self):
        return self.l_dev if self.l_dev is not None else torch.full_like(self.a_dev, self.l_const)

    @property
    def u(self):
        return self.u_dev if self.u_dev is not None else torch.full_like(self.a_dev, self.u_const)

    def __repr__(self):
        return f"BoxLineSet(n={self.n}, d={self.d})"


class ActiveSetMask:
    """Partition into bound-active and free coordinates (ref projection.py:60-79).
    ``free_mask`` is the device 0/1 diagonal of Sigma."""

    def __init__(self, free_mask, v=None, lam=None, box=None):
        self.free_mask = free_mask
        self._v, self._lam, self._box = v, lam, box

    @property
    def free(self):
        return torch.nonzero(self.free_mask, as_tuple=False).flatten()

    @property
    def p(self):
        return int(self.free_mask.sum())

    @property
    def sigma_diag(self):
        return self.free_mask.to(torch.float64)

    def _sides(self):
        y = self._v - self._lam * self._box.a
        l, u = self._box.l, self._box.u
        lower = y <= l + 1e-12 * (1.0 + l.abs())
        upper = (y >= u - 1e-12 * (1.0 + u.abs())) & ~lower
        return lower, upper

    @property
    def lower_active(self):
        return torch.nonzero(self._sides()[0], as_tuple=False).flatten()

    @property
    def upper_active(self):
        return torch.nonzero(self._sides()[1], as_tuple=False).flatten()


class ProjectionResult:
    """Projection, multiplier lambda-hat and active-set mask (ref projection.py:82-105)."""

    __slots__ = ("x", "lambda_hat", "active_mask", "passes", "p_count")

    def __init__(self, x, lambda_hat, active_mask, passes=0, p_count=None):
        self.x = x
        self.lambda_hat = lambda_hat
        self.active_mask = active_mask
        self.passes = passes
        self.p_count = p_count

    def __repr__(self):
        return f"ProjectionResult(lambda_hat={self.lambda_hat}, n={self.x.shape[0]})"


def raise_on_status(status):
    if status == _lib.PROJ_INFEASIBLE_LOW:
        raise InfeasibleProblemError("projection bracket failed below the breakpoint range")
    if status == _lib.PROJ_INFEASIBLE_HIGH:
        raise InfeasibleProblemError("projection bracket failed above the breakpoint range")


def project_box_line(v, box_line):
    """Project ``v`` onto {x : a'x = d, l <= x <= u}; ref projection.py:152-211.

    Returns a ProjectionResult with device tensors ``x`` and ``active_mask.free_mask``
    and the Python float ``lambda_hat``."""
    be = box_line.backend
    v = as_device(v, be)
    if v.dim() != 1 or v.numel() != box_line.n:
        raise InputError(f"expected a vector of length {box_line.n}, got shape {tuple(v.shape)}")
    x = be.empty(box_line.n)
    free = be.empty(box_line.n, torch.uint8)
    states = be.new_states(1)
    st = be.project_sync(v, box_line, states, x_out=x, free_out=free)
    raise_on_status(int(st["status"][0]))
    lam = float(st["lam"][0])
    return ProjectionResult(x, lam, ActiveSetMask(free, v, lam, box_line), int(st["passes"][0]))


def hs_jacobian_apply(mask, a, y):
    """P y without forming P, P = Sigma(I - aa'/(a'Sigma a))Sigma or Sigma;
    ref projection.py:214-225."""
    free = mask.free_mask if isinstance(mask, ActiveSetMask) else mask
    be = default_backend()
    a = as_device(a, be)
    y = as_device(y, be)
    check_vector(y, a.numel(), "hs_jacobian_apply")
    out = be.empty(a.numel())
    be.hs_apply(as_device(free, be, torch.uint8), a, y, 1.0, None, 0.0, out)
    return out
