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
        l_h = np.ascontiguousarray(l.detach().cpu().numpy() if isinstance(l, torch.Tensor) else l,
                                   dtype=np.float64)
        u_h = np.ascontiguousarray(u.detach().cpu().numpy() if isinstance(u, torch.Tensor) else u,
                                   dtype=np.float64)
        if a_h.ndim != 1 or a_h.shape != l_h.shape or a_h.shape != u_h.shape:
            raise InputError("a, l, u must be one-dimensional vectors of equal length")
        if not np.all(l_h < u_h):
            raise InputError("box must satisfy l < u componentwise")
        d = float(d)
        lo = float(np.sum(np.where(a_h > 0, a_h * l_h, a_h * u_h)))
        hi = float(np.sum(np.where(a_h > 0, a_h * u_h, a_h * l_h)))
        slack = 1e-12 * (1.0 + abs(d) + max(abs(lo), abs(hi)))
        if not (lo - slack <= d <= hi + slack):
            raise InfeasibleProblemError(
                f"a'x = {d} unattainable over the box: range is [{lo}, {hi}]")
        self.n = a_h.shape[0]
        self.d = d
        # a_device: the caller's device copy of the same values (e.g. the labels already
        # uploaded for the operator), saving a second upload
        self.a_dev = a_device if a_device is not None else as_device(a_h, self.backend)
        l_uniform = bool(l_h.min() == l_h.max())
        u_uniform = bool(u_h.min() == u_h.max())
        self.l_const = float(l_h[0]) if l_uniform else 0.0
        self.u_const = float(u_h[0]) if u_uniform else 0.0
        self.l_dev = None if l_uniform else as_device(l_h, self.backend)
        self.u_dev = None if u_uniform else as_device(u_h, self.backend)
        self._range_lo, self._range_hi = lo, hi

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
