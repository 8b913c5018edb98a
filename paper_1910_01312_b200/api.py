"""Reference-shaped functional pieces of the SsN inner loop, on the device.

The reference package exports these as public functions (ref __init__.py:38-60):
grad_phi / breakpoints (projection.py:108-131), psi_eval / psi_grad (solver.py:136-148),
newton_direction (solver.py:194-289) and line_search (solver.py:292-319).  Here they
take and return CUDA tensors (host arrays are uploaded) and run on the same sm_100a
kernels the solver uses: the projection records of csrc/proj.cu and csrc/dist.cu, the
factor-space Newton system of the engine (Gram + Cholesky or the p x p Woodbury dual),
and the batched trial projections of the Armijo search.  ``alm_solve`` does not call
them (its native driver fuses the same steps); they exist so code written against the
reference's functional API runs unchanged.
"""

import math

import numpy as np
import torch

from . import _lib
from .backend import as_device
from .errors import InputError, LineSearchError
from .projection import ActiveSetMask, ProjectionResult, project_box_line


def grad_phi(lam, v, box_line):
    """d - a' clip(v - lam a, l, u) (ref projection.py:108-116): one device reduction
    (the shard-local projection record of csrc/dist.cu, mode 0)."""
    be = box_line.backend
    v = as_device(v, be)
    rec = be.zeros(8)
    be.proj_local(v, box_line, 1, [float(lam)], 0, rec)
    return box_line.d - float(rec[0])


def breakpoints(v, box_line):
    """Sorted kinks (v_i - u_i)/a_i, (v_i - l_i)/a_i over a_i != 0, duplicates kept
    (ref projection.py:119-131).  A utility: the device projection never sorts."""
    be = box_line.backend
    v = as_device(v, be)
    a = box_line.a_dev
    nz = a != 0.0
    an, vn = a[nz], v[nz]
    t = torch.cat([(vn - box_line.u[nz]) / an, (vn - box_line.l[nz]) / an])
    return torch.sort(t).values


def _u_of(w_qw_state, problem):
    qw, state = w_qw_state
    be = problem.backend
    u = be.empty(problem.n)
    be.vec(0, -float(state.sigma), as_device(state.x, be), as_device(qw, be), problem.c, u)
    return u


def _psi_from(w, qw, u, proj, state):
    """psi^k(w) = 1/2 w'Qw + (|u|^2 - |u - Pi(u)|^2 - |x|^2) / (2 sigma) (ref
    solver.py:130-133), the norm difference as sum Pi(2u - Pi)."""
    be = proj.x.device
    del be
    sig = float(state.sigma)
    wqw = float(torch.dot(w, qw))
    diff = float(torch.dot(proj.x, 2.0 * u - proj.x))
    x = state.x if isinstance(state.x, torch.Tensor) else torch.as_tensor(state.x)
    x_sq = float(torch.dot(x.to(u.device, torch.float64), x.to(u.device, torch.float64)))
    return 0.5 * wqw + diff / (2.0 * sig) - x_sq / (2.0 * sig)


def psi_eval(w, qw, state, problem):
    """Inner objective psi(w) with one projection (ref solver.py:136-140)."""
    be = problem.backend
    w, qw = as_device(w, be), as_device(qw, be)
    u = _u_of((qw, state), problem)
    proj = project_box_line(u, problem.constraint)
    return _psi_from(w, qw, u, proj, state)


def psi_grad(w, qw, state, problem):
    """Gradient Q(w - Pi(u(w))) and the projection (ref solver.py:143-148)."""
    be = problem.backend
    w, qw = as_device(w, be), as_device(qw, be)
    u = _u_of((qw, state), problem)
    proj = project_box_line(u, problem.constraint)
    s = w - proj.x
    return problem.q_op.matvec(s), proj


def newton_direction(s, grad, proj, sigma, problem, opts):
    """Semismooth Newton direction (ref solver.py:194-289): returns (direction, q_dir,
    dir_q_dir) with q_dir = Q direction.  Solved in factor space:
    t = X^T d from the q x q system I + sigma X_J^T P X_J (Gram + Cholesky) or, when
    p < q, its p x p Woodbury dual; Qd = X t, d'Qd = |t|^2, d = -s - sigma P(Qd)."""
    be = problem.backend
    eng = problem.engine()
    eng._direct_limit = opts.direct_solve_threshold
    s, grad = as_device(s, be), as_device(grad, be)
    free = proj.active_mask.free_mask if isinstance(proj, ProjectionResult) else proj
    free = as_device(free, be, torch.uint8)
    eng.s.copy_(s)
    eng.grad.copy_(grad)
    eng.free.copy_(free)
    eng.w = be.zeros(problem.n)   # the fused dots read w, Qw: none needed here
    eng.qw = be.zeros(problem.n)
    problem.q_op.xt([s], eng.gr[0:1])  # X^T s: the q-space right-hand side
    a = problem.constraint.a_dev
    be.dots([(a, a)], eng.scal[5:6], mask=free)
    p = int(free.sum())
    sc, _ = eng.fetch()
    asa = float(sc[5])
    eng.asa_dev.fill_(asa)
    eng.direction(p, float(sigma), asa)
    sc, _ = eng.fetch(info=p > 0)
    if p > 0 and int(eng.h_info[0]) != 0:
        raise LineSearchError("reduced Newton matrix not SPD")
    return eng.dir.clone(), eng.qdir.clone(), float(sc[3])


def line_search(w, qw, direction, q_dir, dir_q_dir, grad, psi_at_w, u, state, problem, opts):
    """Armijo backtracking along a descent direction (ref solver.py:292-319): one
    projection per trial, evaluated in device batches of ``line_search_batch`` step
    lengths (one host read per batch).  Returns (alpha, w_new, qw_new, psi_new, u_new,
    proj_new)."""
    be = problem.backend
    w, qw, d, qd = (as_device(v, be) for v in (w, qw, direction, q_dir))
    grad, u = as_device(grad, be), as_device(u, be)
    gd = float(torch.dot(grad, d))
    if gd >= 0.0:
        raise LineSearchError(f"not a descent direction (g'd = {gd:.3e})")
    sigma = float(state.sigma)
    x = as_device(state.x, be)
    x_sq = float(torch.dot(x, x))
    w_qw, w_qd = float(torch.dot(w, qw)), float(torch.dot(w, qd))
    box = problem.constraint
    T = max(1, min(int(getattr(opts, "line_search_batch", 8)), 8))
    states = be.new_states(T)
    xo, fo = be.empty((T, problem.n)), be.empty((T, problem.n), torch.uint8)
    alpha, tried = 1.0, 0
    while tried < 61:
        Tb = min(T, 61 - tried)
        alphas = [alpha * opts.backtrack ** k for k in range(Tb)]
        st = be.project_sync(u, box, states, T=Tb, B=qd, coefs=[sigma * a for a in alphas],
                             x_out=xo, free_out=fo)
        for k, a in enumerate(alphas):
            quad = w_qw + 2.0 * a * w_qd + a * a * float(dir_q_dir)
            psi_t = 0.5 * quad + float(st["sum_xv"][k]) / (2.0 * sigma) - x_sq / (2.0 * sigma)
            if psi_t <= psi_at_w + opts.mu * a * gd:
                u_t = u - (sigma * a) * qd
                lam = float(st["lam"][k])
                proj = ProjectionResult(xo[k].clone(), lam,
                                        ActiveSetMask(fo[k].clone(), u_t, lam, box),
                                        int(st["passes"][k]))
                return a, w + a * d, qw + a * qd, psi_t, u_t, proj
        alpha *= opts.backtrack ** Tb
        tried += Tb
    raise LineSearchError("Armijo backtracking exceeded 60 halvings")


__all__ = ["grad_phi", "breakpoints", "psi_eval", "psi_grad", "newton_direction",
           "line_search"]

del math, np, _lib, InputError
