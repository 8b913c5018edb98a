"""SSsNAL solver: augmented Lagrangian outer loop (Algorithm 1) with the sparse
semismooth Newton inner loop (Algorithm 3), device resident.

Mirrors ref solver.py (QpProblem :34-70, AlmOptions :73-84, SsnOptions :87-97,
SolverState :100-110, SolveReport :113-127, psi_eval :136, psi_grad :143,
newton_direction :194-289, line_search :292-319, ssn_solve :331-411,
kkt_residual :414-426, alm_solve :429-530): same control flow, constants,
stopping rules, safeguards and report fields.

What differs is WHERE the arithmetic happens and one algebraic identity:
the reduced Newton system is solved in factor space.  With Q = X X^T,
(Q + sigma Q P Q) d = -Q s has the unique Q-image Q d = X t where

    (I_q + sigma X_J^T (I - a_J a_J^T / a_J^T a_J) X_J) t = -X^T s,

the q x q SPD system of the paper's Prop. 3.5 proof (I_r + sigma L^T Sigma(...)
Sigma L, with L = X).  Q d = X t and d'Qd = ||t||^2 are exactly the two
quantities the reference's p x p system produces (ref solver.py:260-268), and
the same direction representative d = -s - sigma P(Qd) is used (:269).  The
system is SPD for every sigma, so the reference's sigma nudge for a
vanishing denominator (:239-242) is never needed.
"""

import logging
import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .backend import F64, as_device, check_vector
from .errors import InputError, InternalError, LineSearchError
from .projection import ActiveSetMask, BoxLineSet, ProjectionResult, raise_on_status

logger = logging.getLogger("ssnal")


def _half_powers(k):
    return 0.5 ** k


@dataclass
class AlmOptions:
    """Outer-loop controls (ref solver.py:73-84); tolerance sequences summable."""

    sigma0: float = 1.0
    sigma_growth: float = 5.0
    sigma_max: float = 1e8
    tol_kkt: float = 1e-3
    eps_seq: callable = field(default=_half_powers)
    delta_seq: callable = field(default=_half_powers)
    lambda_min_surrogate: float = 1.0
    max_outer: int = 200


@dataclass
class SsnOptions:
    """Inner Newton controls (ref solver.py:87-97).  ``direct_solve_threshold`` and
    ``cg_max_iters`` keep their meaning for the factor-space system (its order is
    the feature dimension q); ``line_search_batch`` is how many step lengths one
    batched projection launch evaluates after a rejected unit step."""

    mu: float = 1e-4
    backtrack: float = 0.5
    tau: float = 0.5
    eta: float = 1e-2
    max_inner: int = 50
    direct_solve_threshold: int = 2000
    cg_max_iters: int = 500
    line_search_batch: int = 8
    # "delta": Armijo on psi differences (Bregman term fused into the trial projections,
    # no psi-resolution stop); "stable": psi via sum Pi(2u - Pi);
    # "reference": ref solver.py:130-133 term for term
    psi_eval: str = "delta"
    engine: str = "native"    # "native": C++ driver (ssnal_alm_solve_dense); "python": _Engine
    profile: bool = False     # native: CUDA-event time per op class -> problem.op_profile


@dataclass
class SolverState:
    """Per-solve state on the device (ref solver.py:100-110)."""

    x: torch.Tensor
    w: torch.Tensor
    qw: torch.Tensor
    sigma: float
    z: torch.Tensor = None
    outer_iter: int = 0
    inner_iter_total: int = 0


@dataclass
class SolveReport:
    """Outcome of a solve (ref solver.py:113-127)."""

    x_opt: object
    kkt_residual: float
    outer_iters: int
    avg_inner_iters: float
    total_inner_iters: int
    unbounded_support_count: int
    objective: float
    wall_time: float
    converged: bool
    solver: str = "ssnal"
    warnings: list = field(default_factory=list)


class QpProblem:
    """min 1/2 x'Qx + c'x s.t. a'x = d, l <= x <= u (ref solver.py:34-70)."""

    def __init__(self, q_op, c, constraint):
        self.q_op = q_op
        self.constraint = constraint
        self.backend = constraint.backend
        self.c = as_device(c, self.backend)
        if self.c.dim() != 1 or self.c.numel() != constraint.n:
            raise InputError("c length does not match the constraint dimension")
        if getattr(q_op, "n", constraint.n) != constraint.n:
            raise InputError("operator dimension does not match the constraint")
        self._engine = None

    @property
    def n(self):
        return self.constraint.n

    def objective(self, x, qx=None):
        x = as_device(x, self.backend)
        if qx is None:
            qx = self.q_op.matvec(x)
        return 0.5 * float(torch.dot(x, qx)) + float(torch.dot(self.c, x))

    def spot_check(self, seed=0, tol=1e-8):
        """Sampled symmetry / PSD check (ref solver.py:58-70)."""
        rng = np.random.default_rng(seed)
        for _ in range(3):
            v = as_device(rng.standard_normal(self.n), self.backend)
            w = as_device(rng.standard_normal(self.n), self.backend)
            qv, qw = self.q_op.matvec(v), self.q_op.matvec(w)
            vqv, wqw = float(v @ qv), float(w @ qw)
            scale = 1.0 + abs(vqv) + abs(wqw)
            if abs(float(w @ qv) - float(v @ qw)) > tol * scale:
                raise InputError("operator is not symmetric")
            if vqv < -tol * float(v @ v):
                raise InputError("operator is not positive semidefinite")

    def engine(self):
        if self._engine is None:
            self._engine = _Engine(self)
        return self._engine


# state-record field offsets (bytes) for device-scalar views
_OFF = {name: spec[1] for name, spec in _lib.PROJ_STATE_DTYPE.fields.items()}


class _Engine:
    """Device buffers and the kernel sequence of one problem.  Host reads happen
    only at the decision points the reference also branches on."""

    def __init__(self, problem, t_max=8):
        self.pb = problem
        self.op = problem.q_op
        self.box = problem.constraint
        self.be = be = problem.backend
        n, q = problem.n, self.op.q
        self.n, self.q = n, q
        self.t_max = t_max
        e = be.empty
        self.u, self.xp, self.s, self.grad = e(n), e(n), e(n), e(n)
        self.qdir, self.dir, self.tmp, self.qx = e(n), e(n), e(n), e(n)
        self.qwx = e((2, n))
        self.free = be.zeros(n, torch.uint8)
        self.tx = e((t_max, n))
        self.tfree = be.zeros((t_max, n), torch.uint8)
        self.J = be.zeros(n, torch.int32)
        self.pcount = be.zeros(1, torch.int64)
        self.gr = e((2, q))
        self.t = e((1, q))
        self._M = None  # q x q system, allocated on first use (q may be 1e6 for CSR)
        self.m1 = e(q)
        self.scal = be.zeros(16)
        self.info = be.zeros(1, torch.int32)
        self.st_cur = be.new_states(1)
        self.st_trial = be.new_states(t_max)
        self.st_kkt = be.new_states(1)
        self.h_scal = be.host_buffer(16, F64)
        self.h_info = be.host_buffer(1, torch.int32)
        self.h_st = be.host_buffer((t_max, _lib.PROJ_STATE_DTYPE.itemsize), torch.uint8)
        self.c_norm = float(torch.linalg.vector_norm(problem.c))
        self.asa_dev = self.st_cur[0, _OFF["sum_a2_free"]:_OFF["sum_a2_free"] + 8].view(F64)
        self.counters = {"projections": 0, "proj_trials": 0, "newton": 0, "syncs": 0}
        self._direct_limit = 2000
        self.line_search_batch = 8  # set from SsnOptions by ssn_solve
        self.backtrack = 0.5
        self.lam_kkt = 0.0  # warm starts for the multiplier search
        self.lam_cur = 0.0

    @property
    def M(self):
        if self._M is None:
            self._M = self.be.empty((self.q, self.q))
        return self._M

    # ------------------------------------------------------------ host reads
    def fetch(self, states=None, T=1, info=False):
        """Copy scalars (+ T state records) to pinned host memory, one stream sync."""
        self.h_scal.copy_(self.scal, non_blocking=True)
        if info:
            self.h_info.copy_(self.info, non_blocking=True)
        if states is not None:
            self.h_st[:T].copy_(states[:T], non_blocking=True)
        self.be.synchronize()
        self.counters["syncs"] += 1
        sc = self.h_scal.numpy().copy()
        st = self.be.read_states(self.h_st[:T]).copy() if states is not None else None
        return sc, st

    def _trial_base(self, B):
        """Line-search trials in the 'delta' psi mode carry the Bregman term against the
        base projection Pi(u) = self.xp (csrc/proj.cu bregman_term)."""
        if B is not None and getattr(self, "psi_delta", False):
            return {"base": self.xp, "base_lam": self.lam_cur}
        return {}

    def _project(self, A, states, T=1, B=None, coefs=None, x_out=None, free_out=None, ref=None,
                 hint=0.0):
        self.be.project(A, self.box, states, T, B, coefs, x_out, free_out, ref, hint=hint,
                        **self._trial_base(B))
        self.counters["projections"] += 1
        self.counters["proj_trials"] += T

    def _finish_states(self, st, states, T, A, B=None, coefs=None, x_out=None, free_out=None,
                       ref=None):
        """Rarely a trial needs more bracketing passes than the default launch."""
        rounds = 0
        while np.all(st["status"] >= 0) and np.any(st["status"] != _lib.PROJ_APPLIED):
            rounds += 1
            self.counters["extra_rounds"] = self.counters.get("extra_rounds", 0) + 1
            if rounds > 20:
                raise InternalError("projection failed to bracket the multiplier")
            self.be.project(A, self.box, states, T, B, coefs, x_out, free_out, ref,
                            phases=_lib.PHASE_EXACT | _lib.PHASE_APPLY, passes=8, newton=0,
                            **self._trial_base(B))
            _, st = self.fetch(states, T)
        for s in st["status"]:
            raise_on_status(int(s))
        return st

    # ------------------------------------------------------------ outer pieces
    def kkt_and_refresh(self, x, w, qw_out=None):
        """R_KKT(x) (ref solver.py:420-426) and, fused into the same two passes
        over X, the outer refresh Qw (ref solver.py:498).  Returns
        (residual, p, objective); leaves Qx in self.qx."""
        op, be = self.op, self.be
        if qw_out is not None:
            g = op.xt([x, w], self.gr)
            op.x(g, self.qwx, k=2)
            self.qx.copy_(self.qwx[0])
            qw_out.copy_(self.qwx[1])
        else:
            g = op.xt([x], self.gr[:1])
            op.x(g, self.qx.view(1, -1), k=1)
        be.vec(1, 0.0, x, self.qx, self.pb.c, self.tmp)  # x - Qx - c
        self._project(self.tmp, self.st_kkt, ref=x, hint=self.lam_kkt)
        be.dots([(x, None), (x, self.qx), (self.pb.c, x)], self.scal)
        sc, st = self.fetch(self.st_kkt)
        st = self._finish_states(st, self.st_kkt, 1, self.tmp, ref=x)
        self.lam_kkt = float(st["lam"][0])
        res = math.sqrt(float(st["sum_dref2"][0])) / (1.0 + math.sqrt(sc[0]))
        obj = 0.5 * sc[1] + sc[2]
        return res, int(st["nfree"][0]), obj

    # ------------------------------------------------------------ inner pieces
    def gradient(self, g2=None):
        """s = w - Pi(u); grad = Q s = X (X^T s); g_r = X^T s kept for the solve; with
        ``g2`` (a device slot) also ||grad||^2 -- one fused library call, as the driver."""
        op, be = self.op, self.be
        be.dense_gradient(op, self.w, self.xp, self.s, self.gr[0], self.grad,
                          g2 if g2 is not None else self.scal[15:16])

    def start_inner(self, x, w, qw, sigma):
        """u = x - sigma (Qw + c), its projection, s and grad (ref solver.py:343-348)."""
        self.x, self.w, self.qw = x, w, qw
        self.sigma = sigma
        be = self.be
        be.vec(0, -sigma, x, qw, self.pb.c, self.u)
        self._project(self.u, self.st_cur, x_out=self.xp, free_out=self.free, ref=x,
                      hint=self.lam_cur)
        self.gradient()
        be.dots([(self.grad, None), (x, None)], self.scal)
        sc, st = self.fetch(self.st_cur)
        if st["status"][0] != _lib.PROJ_APPLIED:  # needed extra passes: redo what used xp
            st = self._finish_states(st, self.st_cur, 1, self.u, x_out=self.xp,
                                     free_out=self.free, ref=x)
            self.gradient()
            be.dots([(self.grad, None), (x, None)], self.scal)
            sc, _ = self.fetch()
        self.lam_cur = float(st["lam"][0])
        return sc, st[0]

    def direction(self, p, sigma, asa=0.0):
        """Newton direction in factor space.  Fills self.dir, self.qdir and queues
        the dots [g'd, w'Qw, w'Qd, d'Qd]; returns nothing (caller fetches)."""
        be, op = self.be, self.op
        if p == 0:  # Sigma = 0: P = 0, d = -s, Qd = -grad (ref solver.py:221-222)
            be.vec(4, -1.0, self.s, None, None, self.dir)
            be.vec(4, -1.0, self.grad, None, None, self.qdir)
            be.dots([(self.grad, self.dir), (self.w, self.qw), (self.w, self.qdir),
                     (self.s, self.grad)], self.scal)
            return
        be.compact(self.free, self.J, self.pcount)
        if p < self.q:  # sample-space p x p system (Woodbury dual), cheaper when p < q
            if p > self.pb_direct_limit():
                raise InternalError("p x p system larger than direct_solve_threshold; "
                                    "the CG path is not built for dense operators")
            be.newton_pspace(op, self.J, p, self.grad, self.box.a_dev, sigma, asa,
                             self.gr[0], self.t[0], self.info)
        else:           # factor-space q x q system
            if self.q > self.pb_direct_limit():
                raise InternalError("q x q system larger than direct_solve_threshold; "
                                    "the CG path is not built for dense operators")
            be.dense_gram(op, self.J, self.pcount, self.n, self.box.a_dev, sigma, self.asa_dev,
                          self.M, self.m1)
            be.chol_solve(self.M, self.q, self.gr[0], -1.0, self.t[0], self.info)
        # Qd = X t, d = -s - sigma P(Qd) (ref solver.py:269), {g'd, w'Qw, w'Qd, t't}: one
        # fused library call (a_J'a_J from the projection record), as the C++ driver
        be.direction_epilogue(op, self.t[0], self.qdir, self.free, self.box.a_dev, self.asa_dev,
                              self.s, sigma, self.grad, self.w, self.qw, self.dir, self.scal[0:4])

    def pb_direct_limit(self):
        return self._direct_limit

    def steepest(self):
        """d = -grad, Qd = Q(-grad) (ref solver.py:367-372)."""
        be, op = self.be, self.op
        be.vec(4, -1.0, self.grad, None, None, self.dir)
        op.xt([self.dir], self.gr[1:2])
        op.x(self.gr[1:2], self.qdir.view(1, -1), k=1)
        be.dots([(self.grad, self.dir), (self.w, self.qw), (self.w, self.qdir),
                 (self.dir, self.qdir)], self.scal)
        sc, _ = self.fetch()
        return sc

    def first_batch_size(self):
        return min(self.t_max, max(1, self.line_search_batch))

    def enqueue_unit_trial(self):
        """Projections of u - sigma*alpha*Qd for the first Armijo batch alpha = 1, beta, ...
        (speculative, enqueued with the direction: one host round trip per Newton step
        in the common case), as the C++ driver."""
        T0 = self.first_batch_size()
        coefs, alpha = [], 1.0
        for _ in range(T0):
            coefs.append(self.sigma * alpha)
            alpha *= self.backtrack
        self._project(self.u, self.st_trial, T0, B=self.qdir, coefs=coefs,
                      x_out=self.tx, free_out=self.tfree, ref=self.x, hint=self.lam_cur)
        return coefs

    def advance(self, p, asa, sigma, with_gradient=True):
        """Pipelined Newton step: [s, grad = Q s, ||grad||^2] + direction at the current
        point + the alpha = 1 trial projection, all enqueued, then ONE host sync.
        Returns (||grad||^2, [g'd, w'Qw, w'Qd, d'Qd], trial-0 record)."""
        if with_gradient:
            self.gradient(self.scal[4:5])
        self.direction(p, sigma, asa)
        coefs = self.enqueue_unit_trial()
        T0 = len(coefs)
        sc, st = self.fetch(self.st_trial, T0, info=(p > 0))
        if p > 0 and int(self.h_info[0]) != 0:
            raise InternalError(f"reduced Newton matrix not SPD (column {int(self.h_info[0])})")
        st = self._finish_states(st, self.st_trial, T0, self.u, B=self.qdir, coefs=coefs,
                                 x_out=self.tx, free_out=self.tfree, ref=self.x)
        return float(sc[4]), [float(v) for v in sc[:4]], st

    def line_search(self, gd, psi0, wqw, wqdir, dqd, x_sq, opts, first=None):
        """Armijo backtracking (ref solver.py:292-319), step lengths evaluated in
        batched projections: alpha = 1 first (``first``: its already computed
        record), then `line_search_batch` at a time.
        Returns (alpha, trial index, state record)."""
        if gd >= 0.0:
            raise LineSearchError(f"not a descent direction (g'd = {gd:.3e})")
        sigma = self.sigma
        alpha = 1.0
        tried = 0
        while tried < 61:
            if tried == 0:
                T = len(first) if first is not None else 1
            else:
                T = min(self.t_max, max(1, opts.line_search_batch), 61 - tried)
            alphas = []
            for _ in range(T):
                alphas.append(alpha)
                alpha *= opts.backtrack
            coefs = [sigma * a for a in alphas]
            if tried == 0 and first is not None:
                st = first
            else:
                self._project(self.u, self.st_trial, T, B=self.qdir, coefs=coefs, x_out=self.tx,
                              free_out=self.tfree, ref=self.x, hint=self.lam_cur)
                _, st = self.fetch(self.st_trial, T)
                st = self._finish_states(st, self.st_trial, T, self.u, B=self.qdir,
                                         coefs=coefs, x_out=self.tx, free_out=self.tfree,
                                         ref=self.x)
            for j, a in enumerate(alphas):
                if opts.psi_eval == "delta":
                    # psi(w + a d) - psi(w) = a g'd + a^2 d'Qd / 2 + B_h / sigma
                    dpsi = a * gd + 0.5 * a * a * dqd + float(st[j]["sum_bh"]) / sigma
                    psi_t = psi0 + dpsi
                    ok = dpsi <= opts.mu * a * gd
                else:
                    quad = wqw + 2.0 * a * wqdir + a * a * dqd
                    psi_t = _psi(quad, st[j], x_sq, sigma, opts.psi_eval)
                    ok = psi_t <= psi0 + opts.mu * a * gd
                if ok:
                    self.lam_cur = float(st["lam"][j])
                    return a, j, st[j], psi_t
            tried += T
        raise LineSearchError("Armijo backtracking exceeded 60 halvings")

    def accept(self, alpha, j):
        """w += alpha d, Qw += alpha Qd, u = u - sigma alpha Qd, Pi(u) from trial j."""
        be = self.be
        be.vec(2, alpha, self.w, self.dir, None, self.w)
        be.vec(2, alpha, self.qw, self.qdir, None, self.qw)
        be.vec(2, -(self.sigma * alpha), self.u, self.qdir, None, self.u)
        self.xp.copy_(self.tx[j])
        self.free.copy_(self.tfree[j])
        self.st_cur.copy_(self.st_trial[j:j + 1])


def _psi(wqw, rec, x_sq, sigma, mode="stable"):
    """psi^k(w) of ref solver.py:130-133 from the projection's fused sums.

    'reference' forms ||u||^2 - ||u - Pi(u)||^2 as the difference of two sums,
    exactly as the reference; its rounding error ~ eps ||u||^2 / sigma swamps the
    Armijo decrease once ||u|| >> ||Pi(u)|| (config 1 stalls at R_KKT 3.7e-6).
    'stable' uses the identical quantity sum Pi(u)_i (2 u_i - Pi(u)_i)."""
    if mode == "reference":
        diff = float(rec["sum_v2"]) - float(rec["sum_r2"])
    else:
        diff = float(rec["sum_xv"])
    return 0.5 * wqw + diff / (2.0 * sigma) - x_sq / (2.0 * sigma)


@dataclass
class _InnerResult:
    u: torch.Tensor
    proj: object
    iterations: int
    converged: bool
    hit_max_inner: bool


def ssn_solve(state, problem, alm_opts, ssn_opts, eps_k, delta_k, trace=None):
    """Inner semismooth Newton solver (ref solver.py:331-411); same criteria (A')/(B'),
    floors and rescue branches.  Mutates state.w / state.qw."""
    eng = problem.engine()
    eng._direct_limit = ssn_opts.direct_solve_threshold
    eng.line_search_batch = ssn_opts.line_search_batch
    eng.backtrack = ssn_opts.backtrack
    eng.cg_eta, eng.cg_tau, eng.cg_max_iters = ssn_opts.eta, ssn_opts.tau, ssn_opts.cg_max_iters
    delta = ssn_opts.psi_eval == "delta"
    eng.psi_delta = delta
    sigma = state.sigma
    coeff = math.sqrt(alm_opts.lambda_min_surrogate / sigma)
    grad_floor = 1e-12 * (1.0 + eng.c_norm)
    sc, cur = eng.start_inner(state.x, state.w, state.qw, sigma)
    x_sq = float(sc[1])
    gnorm2 = float(sc[0])
    converged = False
    exhausted = True
    iterations = 0
    # pipelined: the Newton direction and the unit-step trial of the CURRENT point are
    # computed speculatively together with its gradient (one host sync per step); at
    # the step that meets the stopping test they are simply discarded.
    _, dots, trial0 = eng.advance(int(cur["nfree"]), float(cur["sum_a2_free"]), sigma,
                                  with_gradient=False)
    for _ in range(ssn_opts.max_inner):
        gnorm = math.sqrt(gnorm2)
        if trace is not None:
            trace.append(gnorm)
        dist = math.sqrt(float(cur["sum_dref2"]))
        if gnorm <= coeff * eps_k and gnorm <= coeff * delta_k * dist:
            converged, exhausted = True, False
            break
        if gnorm <= grad_floor:
            converged, exhausted = True, False
            break
        gd, wqw, wqdir, dqd = dots
        eng.counters["newton"] += 1
        steepest = False
        first = trial0
        if gd >= 0.0:
            sc = eng.steepest()
            gd, wqw, wqdir, dqd = (float(v) for v in sc[:4])
            steepest = True
            first = None
        psi0 = _psi(wqw, cur, x_sq, sigma, ssn_opts.psi_eval)
        # predicted decrease below the resolution of psi (ref solver.py:369-371); the
        # 'delta' mode forms psi differences directly and has no such floor
        if not delta and ssn_opts.mu * abs(gd) <= 1e-16 * (1.0 + abs(psi0)):
            converged, exhausted = True, False
            break
        try:
            alpha, j, cur, _ = eng.line_search(gd, psi0, wqw, wqdir, dqd, x_sq, ssn_opts,
                                               first=first)
        except LineSearchError:
            if steepest:
                exhausted = False
                break
            sc = eng.steepest()
            gd, wqw, wqdir, dqd = (float(v) for v in sc[:4])
            if not delta and ssn_opts.mu * (-gd) <= 1e-16 * (1.0 + abs(psi0)):
                exhausted = False
                break
            try:
                alpha, j, cur, _ = eng.line_search(gd, psi0, wqw, wqdir, dqd, x_sq, ssn_opts)
            except LineSearchError:
                exhausted = False
                break
        eng.accept(alpha, j)
        iterations += 1
        gnorm2, dots, trial0 = eng.advance(int(cur["nfree"]), float(cur["sum_a2_free"]), sigma)
    if exhausted and trace is not None:
        trace.append(math.sqrt(gnorm2))
    state.inner_iter_total += iterations
    lam = float(cur["lam"])
    proj = ProjectionResult(eng.xp, lam, ActiveSetMask(eng.free, eng.u, lam, eng.box))
    proj.p_count = int(cur["nfree"])
    return _InnerResult(eng.u, proj, iterations, converged, exhausted)


def kkt_residual(x, problem):
    """||x - Pi(x - Qx - c)|| / (1 + ||x||) (ref solver.py:414-417)."""
    x = as_device(x, problem.backend)
    check_vector(x, problem.n, "kkt_residual")
    return problem.engine().kkt_and_refresh(x, None)[0]


def _native_ok(problem, alm_opts, ssn_opts):
    from .operators import CsrKernelOperator, LinearKernelOperator

    comm = getattr(problem, "comm", None)
    if comm is not None:
        # row-sharded: the native sharded driver over NCCL (ssnal_alm_solve_sharded); gloo
        # groups (CPU tests) and engine="python" run sharded.ShardedEngine
        return (comm.nccl and ssn_opts.engine == "native"
                and isinstance(problem.q_op, (CsrKernelOperator, LinearKernelOperator))
                and alm_opts.eps_seq is _half_powers and alm_opts.delta_seq is _half_powers)
    if isinstance(problem.q_op, CsrKernelOperator):
        if not (alm_opts.eps_seq is _half_powers and alm_opts.delta_seq is _half_powers):
            raise InputError("the sparse operator runs only in the native driver, which uses "
                             "the reference's default eps/delta sequences")
        return True
    return (ssn_opts.engine == "native" and getattr(problem.backend, "name", "") == "cuda"
            and isinstance(problem.q_op, LinearKernelOperator)
            and alm_opts.eps_seq is _half_powers and alm_opts.delta_seq is _half_powers)


_PSI_MODES = {"reference": 0, "stable": 1, "delta": 2}


def _alm_solve_native(problem, alm_opts, ssn_opts, x0, w0, callback, return_device, comm=None):
    """The same loop through the C++ driver (csrc/driver.cu): one C-ABI call.  With
    ``comm`` (a _lib.Comm) the problem is one rank's slice and the row-sharded driver
    (ssnal_alm_solve_sharded) runs it with the other ranks."""
    import ctypes

    be, op, box = problem.backend, problem.q_op, problem.constraint
    n = problem.n
    lib = _lib.load()
    sparse = getattr(op, "kind", "dense") == "csr"
    if comm is not None:
        nbytes = (lib.ssnal_alm_ws_bytes_csr_sharded(op._cref, comm.world) if sparse else
                  lib.ssnal_alm_ws_bytes_sharded(op.n_phys, op.q, int(op.svr_block), comm.world))
    elif sparse:
        nbytes = lib.ssnal_alm_ws_bytes_csr(op._cref)
    else:
        nbytes = lib.ssnal_alm_ws_bytes(op.n_phys, op.q, int(op.svr_block))
    ws = getattr(problem, "_native_ws", None)
    if ws is None or ws.numel() < nbytes:
        ws = be.zeros(int(nbytes), torch.uint8)
        problem._native_ws = ws
    ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
    prob = _lib.DenseProblem(
        A=None if sparse else ptr(op.A), n_phys=op.n_phys, q=op.q, lda=op.lda,
        row_sign=ptr(op.row_sign), svr_block=int(op.svr_block), n=n, c=ptr(problem.c),
        a=ptr(box.a_dev), l=ptr(box.l_dev), u=ptr(box.u_dev), l_const=box.l_const,
        u_const=box.u_const, d=float(getattr(box, "d_global", box.d)), csr=ctypes.pointer(op.c_op) if sparse else None)
    opts = _lib.Options(
        sigma0=alm_opts.sigma0, sigma_growth=alm_opts.sigma_growth, sigma_max=alm_opts.sigma_max,
        tol_kkt=alm_opts.tol_kkt, lambda_min_surrogate=alm_opts.lambda_min_surrogate,
        max_outer=alm_opts.max_outer, mu=ssn_opts.mu, backtrack=ssn_opts.backtrack,
        tau=ssn_opts.tau, eta=ssn_opts.eta, max_inner=ssn_opts.max_inner,
        direct_solve_threshold=ssn_opts.direct_solve_threshold,
        cg_max_iters=ssn_opts.cg_max_iters, line_search_batch=ssn_opts.line_search_batch,
        psi_stable=_PSI_MODES[ssn_opts.psi_eval], profile=int(bool(ssn_opts.profile)))
    x0d = None if x0 is None else as_device(x0, be)
    w0d = None if w0 is None else as_device(w0, be)
    if x0d is not None:
        check_vector(x0d, n, "x0")
    if w0d is not None:
        check_vector(w0d, n, "w0")
    x_out = be.empty(n)
    rep = _lib.Report()
    if callback is not None:
        cb = _lib.PROGRESS_FN(lambda k, r, s, p, inner, ctx: callback(k, r, s, int(p), inner))
    else:
        cb = _lib.PROGRESS_FN()
    if comm is None:
        _lib.call("ssnal_alm_solve_dense", ctypes.byref(prob), ctypes.byref(opts), ptr(x0d),
                  ptr(w0d), ptr(x_out), ctypes.byref(rep), ptr(ws), ws.numel(), cb, None,
                  be.stream())
    else:
        _lib.call("ssnal_alm_solve_sharded", ctypes.byref(prob), ctypes.byref(opts),
                  ctypes.byref(comm), ptr(x0d), ptr(w0d), ptr(x_out), ctypes.byref(rep), ptr(ws),
                  ws.numel(), cb, None, be.stream())
    notes = [f"inner solver hit max_inner at outer iteration {k}" for k in range(64)
             if rep.hit_max_inner_mask64 >> k & 1]
    if rep.hit_max_inner_count > len(notes):
        notes.append(f"inner solver hit max_inner at {rep.hit_max_inner_count - len(notes)} "
                     "more outer iterations (k >= 64)")
    if rep.stagnated:
        notes.append("stagnated at the attainable accuracy for sigma_max; returning the best "
                     "iterate")
    if rep.max_outer_reached:
        notes.append(f"max_outer={alm_opts.max_outer} reached")
    problem.native_counters = {"syncs": rep.syncs, "newton": rep.newton_steps,
                               "projections": rep.projections, "cg_iters": rep.cg_iters,
                               "cg_fallbacks": rep.cg_fallbacks,
                               "gram_builds": rep.gram_builds, "gram_updates": rep.gram_updates,
                               "gram_rows": rep.gram_rows, "proj_fallbacks": rep.proj_fallbacks}
    problem.op_profile = {name: {"calls": int(rep.op_calls[k]), "seconds": float(rep.op_seconds[k]),
                                 "bytes": float(rep.op_bytes[k]), "flops": float(rep.op_flops[k])}
                          for k, name in enumerate(_lib.OP_NAMES)}
    return SolveReport(
        x_opt=x_out if return_device else x_out.cpu().numpy(),
        kkt_residual=rep.kkt_residual, outer_iters=rep.outer_iters,
        avg_inner_iters=rep.total_inner_iters / max(rep.outer_iters, 1),
        total_inner_iters=rep.total_inner_iters,
        unbounded_support_count=rep.unbounded_support_count, objective=rep.objective,
        wall_time=rep.wall_time, converged=bool(rep.converged), solver="ssnal", warnings=notes)


def alm_solve(problem, alm_opts=None, ssn_opts=None, x0=None, w0=None, callback=None,
              return_device=False):
    """SSsNAL (ref solver.py:429-530).  Inputs may be host arrays; ``x_opt`` is
    returned as a numpy array (device tensor with ``return_device=True``).

    Runs in the native C++ driver (one C-ABI call, csrc/driver.cu) when possible,
    else in the Python mirror below (same control flow; used for custom tolerance
    sequences, the test backends and the sharded path)."""
    alm_opts = alm_opts or AlmOptions()
    ssn_opts = ssn_opts or SsnOptions()
    if _native_ok(problem, alm_opts, ssn_opts):
        comm = getattr(problem, "comm", None)
        return _alm_solve_native(problem, alm_opts, ssn_opts, x0, w0, callback, return_device,
                                 comm=None if comm is None else comm.native())
    t_start = time.perf_counter()
    eng = problem.engine()
    eng._direct_limit = ssn_opts.direct_solve_threshold
    be = problem.backend
    n = problem.n
    x = be.zeros(n) if x0 is None else as_device(x0, be).clone()
    w = be.zeros(n) if w0 is None else as_device(w0, be).clone()
    if x0 is not None:
        check_vector(x, n, "x0")
    if w0 is not None:
        check_vector(w, n, "w0")
    qw = be.zeros(n)
    state = SolverState(x=x, w=w, qw=qw, sigma=alm_opts.sigma0)

    warnings_out = []
    converged = False
    inner_last = 0
    p_last = None
    residual = math.inf
    obj_last = None
    outer = 0
    best = None
    stalled = 0
    for k in range(alm_opts.max_outer + 1):
        residual, p_kkt, obj_last = eng.kkt_and_refresh(state.x, state.w, state.qw)
        if p_last is None:
            p_last = p_kkt
        logger.info("outer=%d rkkt=%.3e sigma=%.2e p=%d inner=%d",
                    k, residual, state.sigma, p_last, inner_last)
        if callback is not None:
            callback(k, residual, state.sigma, p_last, inner_last)
        if best is None or residual < best[0]:
            best = (residual, state.x, p_last, obj_last)
            stalled = 0
        elif state.sigma >= alm_opts.sigma_max:
            stalled += 1
            if stalled >= 3:
                warnings_out.append("stagnated at the attainable accuracy for sigma_max; "
                                    "returning the best iterate")
                break
        if residual < alm_opts.tol_kkt:
            converged = True
            break
        if k == alm_opts.max_outer:
            warnings_out.append(f"max_outer={alm_opts.max_outer} reached")
            break
        inner = ssn_solve(state, problem, alm_opts, ssn_opts,
                          eps_k=alm_opts.eps_seq(k), delta_k=alm_opts.delta_seq(k))
        if inner.hit_max_inner:
            warnings_out.append(f"inner solver hit max_inner at outer iteration {k}")
        state.x = inner.proj.x.clone()
        p_last = inner.proj.p_count
        inner_last = inner.iterations
        state.sigma = min(state.sigma * alm_opts.sigma_growth, alm_opts.sigma_max)
        state.outer_iter += 1
        outer += 1

    if best is not None and best[0] < residual:
        residual, x_ret, p_ret, objective = best
    else:
        x_ret, p_ret, objective = state.x, p_last, obj_last
    return SolveReport(
        x_opt=x_ret if return_device else x_ret.cpu().numpy(),
        kkt_residual=residual,
        outer_iters=outer,
        avg_inner_iters=state.inner_iter_total / max(outer, 1),
        total_inner_iters=state.inner_iter_total,
        unbounded_support_count=int(p_ret),
        objective=objective,
        wall_time=time.perf_counter() - t_start,
        converged=converged,
        solver="ssnal",
        warnings=warnings_out,
    )
