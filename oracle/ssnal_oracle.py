"""numpy restatement of the reference SSsNAL path (test infrastructure only).

Every function cites the reference file:line it restates; "ref" below means
``/root/reference/pkg/src/ssnal``.  Two deliberate representation choices,
neither of which changes the mathematics:

* the SVM operators are held in factored form Q = X X^T (X = diag(y) A for
  C-SVC, X = [A; -A] for SVR), so ``matvec`` costs O(nq) instead of the
  reference's column-by-column O(n^2 q) (ref kernels.py:144-154).  Columns and
  principal submatrices are produced from the factor with the same values;
* the solver returns plain dicts instead of dataclasses.

Numerical branches (sigma nudging, lstsq fallback, CG fallback, steepest
descent rescue, best-iterate safeguard) follow the reference one for one.
"""

import math
import time
import warnings

import numpy as np
import scipy.linalg

__all__ = [
    "BoxLine", "InfeasibleError", "LineSearchFailed",
    "grad_phi", "breakpoints", "classify_free", "project", "hs_apply",
    "DenseQ", "FactoredQ", "SvrFactoredQ", "CsrFactoredQ", "newton_direction_factor",
    "AlmOpts", "SsnOpts", "psi_value", "newton_direction", "line_search",
    "ssn_solve", "kkt_residual", "kkt_full", "alm_solve", "set_psi_mode", "PSI_MODE", "bregman",
    "csvc_problem", "csvc_problem_csr", "svr_problem", "objective",
]

ACTIVE_TOL = 1e-12  # ref projection.py:19


class InfeasibleError(ValueError):
    pass


class LineSearchFailed(RuntimeError):
    pass


class BoxLine:
    """{x : a'x = d, l <= x <= u}; ref projection.py:22-54 (feasibility checked once)."""

    def __init__(self, a, d, l, u):
        self.a = np.ascontiguousarray(a, dtype=np.float64)
        self.l = np.ascontiguousarray(l, dtype=np.float64)
        self.u = np.ascontiguousarray(u, dtype=np.float64)
        self.d = float(d)
        if not (self.a.ndim == 1 and self.a.shape == self.l.shape == self.u.shape):
            raise ValueError("a, l, u must be equal-length vectors")
        if not np.all(self.l < self.u):
            raise ValueError("box must satisfy l < u")
        pos = self.a > 0
        lo = float(np.sum(np.where(pos, self.a * self.l, self.a * self.u)))
        hi = float(np.sum(np.where(pos, self.a * self.u, self.a * self.l)))
        slack = 1e-12 * (1.0 + abs(self.d) + max(abs(lo), abs(hi)))
        if not (lo - slack <= self.d <= hi + slack):
            raise InfeasibleError(f"a'x = {self.d} unattainable; range [{lo}, {hi}]")
        self.n = self.a.size
        self.nz = np.flatnonzero(self.a != 0.0)


def grad_phi(lam, v, s):
    """d - a' clip(v - lam a, l, u); ref projection.py:108-116."""
    return s.d - float(s.a.dot(np.minimum(np.maximum(v - lam * s.a, s.l), s.u)))


def breakpoints(v, s):
    """Sorted kinks (v_i-u_i)/a_i, (v_i-l_i)/a_i over a_i != 0; ref projection.py:119-131."""
    if s.nz.size == 0:
        return np.empty(0)
    an = s.a[s.nz]
    vn = v[s.nz]
    return np.sort(np.concatenate(((vn - s.u[s.nz]) / an, (vn - s.l[s.nz]) / an)))


def classify_free(v, lam, s):
    """Free-set mask of the projection (bound slots get tolerance 1e-12(1+|b|));
    ref projection.py:134-149."""
    y = v - lam * s.a
    lower = y <= s.l + ACTIVE_TOL * (1.0 + np.abs(s.l))
    upper = (y >= s.u - ACTIVE_TOL * (1.0 + np.abs(s.u))) & ~lower
    return ~(lower | upper)


def project(v, s):
    """Breakpoint-search projection onto K cap L.  Returns (x, lambda, free_mask).

    ref projection.py:152-211 (binary search over sorted breakpoints keeping
    grad_phi < 0 on the left, >= 0 on the right; linear interpolation on the
    last segment; lambda = t_l on zero-width brackets).
    """
    v = np.asarray(v, dtype=np.float64)
    if v.shape != (s.n,):
        raise ValueError(f"expected length {s.n}")
    ts = breakpoints(v, s)
    if ts.size == 0:
        lam = 0.0
    else:
        f_first = grad_phi(ts[0], v, s)
        f_last = grad_phi(ts[-1], v, s)
        if f_first >= 0.0:
            if f_first > 1e-9 * (1.0 + abs(s.d)):
                raise InfeasibleError("bracket failed below the breakpoint range")
            lam = float(ts[0])
        elif f_last < 0.0:
            raise InfeasibleError("bracket failed above the breakpoint range")
        else:
            lo, hi, f_lo, f_hi = 0, ts.size - 1, f_first, f_last
            while hi - lo > 1 and ts[hi] > ts[lo]:
                mid = (lo + hi) // 2
                f_mid = grad_phi(ts[mid], v, s)
                if f_mid >= 0.0:
                    hi, f_hi = mid, f_mid
                else:
                    lo, f_lo = mid, f_mid
            if f_hi == f_lo or ts[hi] == ts[lo]:
                lam = float(ts[lo])
            else:
                lam = float(ts[lo] - f_lo * (ts[hi] - ts[lo]) / (f_hi - f_lo))
    x = np.minimum(np.maximum(v - lam * s.a, s.l), s.u)
    return x, lam, classify_free(v, lam, s)


def hs_apply(free, a, y):
    """HS-Jacobian product P y, P = S(I - aa'/(a'Sa))S or S; ref projection.py:214-225."""
    z = np.where(free, y, 0.0)
    af = np.where(free, a, 0.0)
    ss = float(af.dot(af))
    if ss != 0.0:
        z = z - (af.dot(z) / ss) * af
    return z


# --------------------------------------------------------------------------
# Q operators (matvec / columns / submatrix), ref kernels.py:68-238
# --------------------------------------------------------------------------

class DenseQ:
    """Explicit Q; ref kernels.py:218-238."""

    def __init__(self, q):
        self.q = np.ascontiguousarray(q, dtype=np.float64)
        self.n = self.q.shape[0]

    def matvec(self, v):
        return self.q @ v

    def columns(self, idx):
        return self.q[:, idx].copy()  # C-contiguous, as ref kernels.py:230-231

    def submatrix(self, idx):
        return self.q[np.ix_(idx, idx)].copy()


class FactoredQ:
    """Q = X X^T with X = diag(row_sign) A (linear-kernel C-SVC: Q_ij = y_i y_j a_i'a_j,
    the same entries as ref kernels.py:97-106 with a linear KernelSpec)."""

    def __init__(self, a_mat, row_sign=None):
        self.A = np.ascontiguousarray(a_mat, dtype=np.float64)
        self.sign = None if row_sign is None else np.asarray(row_sign, dtype=np.float64)
        self.n = self.A.shape[0]

    def _rows(self, idx):
        r = self.A[idx]
        return r if self.sign is None else self.sign[idx, None] * r

    def xt(self, v):
        return self.A.T @ (v if self.sign is None else self.sign * v)

    def x(self, t):
        r = self.A @ t
        if self.sign is None:
            return r
        return self.sign * r if r.ndim == 1 else self.sign[:, None] * r

    def matvec(self, v):
        return self.x(self.xt(v))

    def rows(self, idx):
        """X_J (p x q): the rows of the factor for the slots idx."""
        return self._rows(np.asarray(idx, dtype=np.int64))

    def columns(self, idx):
        return self.x(self._rows(np.asarray(idx, dtype=np.int64)).T)

    def submatrix(self, idx):
        r = self._rows(np.asarray(idx, dtype=np.int64))
        return r @ r.T


class SvrFactoredQ:
    """Q = [[K,-K],[-K,K]] with K = A A^T, i.e. X = [A; -A]; ref kernels.py:181-215."""

    def __init__(self, a_mat):
        self.A = np.ascontiguousarray(a_mat, dtype=np.float64)
        self.m = self.A.shape[0]
        self.n = 2 * self.m

    def _rows(self, idx):
        idx = np.asarray(idx, dtype=np.int64)
        sgn = np.where(idx < self.m, 1.0, -1.0)
        return sgn[:, None] * self.A[idx % self.m]

    def xt(self, v):
        return self.A.T @ (v[: self.m] - v[self.m:])

    def x(self, t):
        r = self.A @ t
        return np.concatenate([r, -r], axis=0)

    def matvec(self, v):
        return self.x(self.xt(v))

    def rows(self, idx):
        return self._rows(idx)

    def columns(self, idx):
        return self.x(self._rows(idx).T)

    def submatrix(self, idx):
        r = self._rows(idx)
        return r @ r.T


class CsrFactoredQ:
    """Q = X X^T with X = diag(row_sign) A, A a scipy CSR matrix (sparse linear-kernel
    C-SVC; the same Q entries as ref kernels.py:97-106 with sparse sample vectors).
    ``rows`` returns X_J as a CSR matrix; ``submatrix`` the dense p x p Q_JJ."""

    def __init__(self, indptr, indices, data, shape, row_sign=None):
        import scipy.sparse as sp

        self.A = sp.csr_matrix((np.asarray(data, dtype=np.float64), np.asarray(indices),
                                np.asarray(indptr)), shape=shape)
        self.AT = self.A.T.tocsr()
        self.sign = None if row_sign is None else np.asarray(row_sign, dtype=np.float64)
        self.n, self.q = shape

    def xt(self, v):
        return self.AT @ (v if self.sign is None else self.sign * v)

    def x(self, t):
        r = self.A @ t
        return r if self.sign is None else self.sign * r

    def matvec(self, v):
        return self.x(self.xt(v))

    def rows(self, idx):
        import scipy.sparse as sp

        idx = np.asarray(idx, dtype=np.int64)
        r = self.A[idx]
        return r if self.sign is None else sp.diags(self.sign[idx]) @ r

    def columns(self, idx):
        r = self.rows(idx)
        return np.asarray(self.x(r.T.toarray()))

    def submatrix(self, idx):
        r = self.rows(idx)
        return np.asarray((r @ r.T).toarray())


def csvc_problem_csr(indptr, indices, data, shape, y, C):
    """Sparse C-SVC dual (CSR samples): as csvc_problem; ref svm.py:95-108."""
    y = np.asarray(y, dtype=np.float64)
    n = y.size
    op = CsrFactoredQ(indptr, indices, data, shape, y)
    return op, -np.ones(n), BoxLine(y, 0.0, np.zeros(n), np.full(n, float(C)))


def csvc_problem(a_mat, y, C):
    """C-SVC dual with linear kernel: Q = diag(y)AA^T diag(y), c = -e, a = y, d = 0,
    box [0, C]; ref svm.py:95-108."""
    y = np.asarray(y, dtype=np.float64)
    n = y.size
    return FactoredQ(a_mat, y), -np.ones(n), BoxLine(y, 0.0, np.zeros(n), np.full(n, float(C)))


def svr_problem(a_mat, t, C, eps):
    """eps-SVR dual over 2n variables: c = (eps - t; eps + t), a = (e; -e), d = 0,
    box [0, C]; ref svm.py:111-127."""
    t = np.asarray(t, dtype=np.float64)
    n = t.size
    c = np.concatenate([eps - t, eps + t])
    a = np.concatenate([np.ones(n), -np.ones(n)])
    return SvrFactoredQ(a_mat), c, BoxLine(a, 0.0, np.zeros(2 * n), np.full(2 * n, float(C)))


def objective(op, c, x, qx=None):
    """Primal value 1/2 x'Qx + c'x; ref solver.py:53-56."""
    if qx is None:
        qx = op.matvec(x)
    return 0.5 * float(x.dot(qx)) + float(c.dot(x))


# --------------------------------------------------------------------------
# Solver, ref solver.py
# --------------------------------------------------------------------------

class AlmOpts:
    """ref solver.py:73-84."""

    def __init__(self, sigma0=1.0, sigma_growth=5.0, sigma_max=1e8, tol_kkt=1e-3,
                 lambda_min_surrogate=1.0, max_outer=200):
        self.sigma0 = sigma0
        self.sigma_growth = sigma_growth
        self.sigma_max = sigma_max
        self.tol_kkt = tol_kkt
        self.lambda_min_surrogate = lambda_min_surrogate
        self.max_outer = max_outer

    @staticmethod
    def eps_seq(k):
        return 0.5 ** k

    delta_seq = eps_seq


class SsnOpts:
    """ref solver.py:87-97."""

    def __init__(self, mu=1e-4, backtrack=0.5, tau=0.5, eta=1e-2, max_inner=50,
                 direct_solve_threshold=2000, cg_max_iters=500, newton="reference",
                 cg_eta_cap=1e-4):
        # newton: "reference" = ref solver.py:194-289 (columns of Q, p x p system);
        # "factor" = newton_direction_factor (same direction from the factor X, for
        # problems whose p x n column block does not fit: configs 2-4 at full size)
        self.newton = newton
        self.cg_eta_cap = cg_eta_cap
        self.mu = mu
        self.backtrack = backtrack
        self.tau = tau
        self.eta = eta
        self.max_inner = max_inner
        self.direct_solve_threshold = direct_solve_threshold
        self.cg_max_iters = cg_max_iters


PSI_MODE = {"mode": "reference"}


def set_psi_mode(mode):
    """'reference' (ref solver.py:130-133 verbatim) or 'stable': the same psi with
    ||u||^2 - ||u - Pi(u)||^2 evaluated as Pi(u)'(2u - Pi(u)) -- identical in exact
    arithmetic, free of the cancellation that stalls Armijo when ||u|| >> ||Pi(u)||
    (the product path's evaluation).
    The product's 'delta' mode (line search on psi differences)
    is restated too: psi(w + a d) - psi(w) = a g'd + a^2 d'Qd / 2 + B_h / sigma with
    B_h = sum (x_t - Pi)(u_t - (x_t + Pi)/2 - lam_bar a) the Bregman divergence of
    h = |.|^2/2 - dist(., K)^2/2, and no psi-resolution floor."""
    if mode not in ("reference", "stable", "delta"):
        raise ValueError(mode)
    PSI_MODE["mode"] = mode


def psi_value(w_qw, u, px, x_sq, sigma):
    """ref solver.py:130-133."""
    if PSI_MODE["mode"] in ("stable", "delta"):
        return 0.5 * w_qw + float(px.dot(2.0 * u - px)) / (2.0 * sigma) - x_sq / (2.0 * sigma)
    r = u - px
    return 0.5 * w_qw + (float(u.dot(u)) - float(r.dot(r))) / (2.0 * sigma) - x_sq / (2.0 * sigma)


def _cg(apply_m, rhs, atol, max_iters):
    """ref solver.py:151-172."""
    v = np.zeros_like(rhs)
    r = rhs.copy()
    p = r.copy()
    rs = float(r.dot(r))
    if math.sqrt(rs) <= atol:
        return v, True
    for _ in range(max_iters):
        mp = apply_m(p)
        den = float(p.dot(mp))
        if den <= 0.0:
            return v, False
        step = rs / den
        v += step * p
        r -= step * mp
        rs_new = float(r.dot(r))
        if math.sqrt(rs_new) <= atol:
            return v, True
        p = r + (rs_new / rs) * p
        rs = rs_new
    return v, False


def _solve_sym(m, rhs):
    """Symmetric solve, min-norm lstsq on LinAlgWarning/Error; ref solver.py:175-191."""
    with warnings.catch_warnings(record=True) as caught:
        warnings.simplefilter("always", scipy.linalg.LinAlgWarning)
        try:
            v = scipy.linalg.solve(m, rhs, assume_a="sym")
        except scipy.linalg.LinAlgError:
            return np.linalg.lstsq(m, rhs, rcond=1e-12)[0]
    if any(issubclass(w.category, scipy.linalg.LinAlgWarning) for w in caught):
        return np.linalg.lstsq(m, rhs, rcond=1e-12)[0]
    return v


def newton_direction(s, grad, free, sigma, op, a, opts):
    """Reduced p x p Newton system of Prop. 3.5; ref solver.py:194-289.

    Returns (direction, q_dir, dir_q_dir)."""
    J = np.flatnonzero(free)
    p = J.size
    s_qs = float(s.dot(grad))
    if p == 0:
        return -s.copy(), -grad.copy(), s_qs
    cols = op.columns(J)
    q_jj = cols[J, :]
    g_j = grad[J]
    a_j = a[J]
    target = min(opts.eta, float(np.linalg.norm(grad)) ** (1.0 + opts.tau))
    a_sa = float(a_j.dot(a_j))
    if a_sa != 0.0:
        qa = q_jj @ a_j
        aqa = float(a_j.dot(qa))
        sig = sigma
        den = a_sa - sig * aqa
        scale = a_sa + abs(sig * aqa)
        tries = 0
        while abs(den) <= 1e-12 * scale and tries < 8:
            sig *= 1.0 + 1e-6
            den = a_sa - sig * aqa
            tries += 1
        ag = float(a_j.dot(g_j))
        rhs = g_j + (sig * ag / den) * qa

        def dense_m():
            m = q_jj + (sig / den) * np.outer(qa, qa)
            m[np.diag_indices_from(m)] += 1.0 / sig
            return m

        if p <= opts.direct_solve_threshold:
            v = _solve_sym(dense_m(), rhs)
        else:
            v, ok = _cg(lambda t: t / sig + q_jj @ t + (sig * float(qa.dot(t)) / den) * qa,
                        rhs, target, opts.cg_max_iters)
            if not ok:
                v = _solve_sym(dense_m(), rhs)
        qv = q_jj @ v
        gamma = float(a_j.dot(qv)) - ag
        q_dir = cols @ v - grad + (sig * gamma / den) * (cols @ a_j)
        dqd = (float(v.dot(qv)) - 2.0 * float(v.dot(g_j)) + s_qs
               + (2.0 * sig * a_sa - sig * sig * aqa) / (den * den) * gamma * gamma)
        direction = -s - sig * hs_apply(free, a, q_dir)
    else:
        def dense_m():
            m = q_jj.copy()
            m[np.diag_indices_from(m)] += 1.0 / sigma
            return m

        if p <= opts.direct_solve_threshold:
            v = _solve_sym(dense_m(), g_j)
        else:
            v, ok = _cg(lambda t: t / sigma + q_jj @ t, g_j, target, opts.cg_max_iters)
            if not ok:
                v = _solve_sym(dense_m(), g_j)
        q_dir = cols @ v - grad
        dqd = float(v.dot(q_jj @ v)) - 2.0 * float(v.dot(g_j)) + s_qs
        direction = -s - sigma * hs_apply(free, a, q_dir)
    return direction, q_dir, dqd


def _pcg(apply_m, rhs, dinv, done, max_iters, check_every=10):
    """Jacobi-preconditioned CG from 0; ``done(v)`` is the stopping test, evaluated
    every ``check_every`` iterations.  Returns (v, converged)."""
    v = np.zeros_like(rhs)
    r = rhs.copy()
    z = dinv * r
    p = z.copy()
    rz = float(r.dot(z))
    if not np.any(rhs):
        return v, True
    for it in range(1, max_iters + 1):
        mp = apply_m(p)
        den = float(p.dot(mp))
        if den <= 0.0:
            return v, False
        step = rz / den
        v += step * p
        r -= step * mp
        if it % check_every == 0 and done(v):
            return v, True
        z = dinv * r
        rz_new = float(r.dot(z))
        if rz_new == 0.0:  # exact solution reached
            return v, True
        p = z + (rz_new / rz) * p
        rz = rz_new
    return v, done(v)


def newton_direction_factor(s, grad, free, sigma, op, a, opts):
    """The Newton direction of ref solver.py:194-289 computed from the factor Q = X X^T
     -- the same (d, Qd, d'Qd) up to rounding, without the
    n x p column block the reference forms:

      t = X^T d solves  (I_q + sigma X_J^T P_J X_J) t = -X^T s,  P_J = I - a_J a_J'/a_J'a_J,
      Qd = X t,  d'Qd = |t|^2,  d = -s - sigma P(Qd)  (ref solver.py:269 representative).

    Routes (ref solver.py:238-258 policy on min(p, q)): q <= threshold -> q x q Cholesky;
    p <= threshold -> the Woodbury p x p system (I + sigma P Q_JJ P) y = P g_J,
    t = -X^T s + sigma X_J^T P y; else Jacobi-PCG on the q-space system, stopped on the
    Newton residual |sigma X X_J^T P X_J t + ...| of Algorithm 3 at 1/10 of
    min(cg_eta_cap, |grad|^(1+tau)) (the product's matrix-free tolerance, tighter)."""
    J = np.flatnonzero(free)
    p = J.size
    r = op.xt(s)
    q = r.size
    if p == 0:
        return -s.copy(), -grad.copy(), float(r.dot(r))
    xj = op.rows(J)
    a_j = a[J]
    asa = float(a_j.dot(a_j))
    m1 = np.asarray(xj.T @ a_j).ravel()
    thr = opts.direct_solve_threshold
    if q <= thr:
        g = xj.T @ xj
        g = np.asarray(g.toarray() if hasattr(g, "toarray") else g)
        m = g - np.outer(m1, m1) / asa if asa != 0.0 else g.copy()
        m *= sigma
        m[np.diag_indices_from(m)] += 1.0
        t = -scipy.linalg.cho_solve(scipy.linalg.cho_factor(m, lower=True), r)
    elif p <= thr:
        qjj = xj @ xj.T
        qjj = np.asarray(qjj.toarray() if hasattr(qjj, "toarray") else qjj)
        g_j = grad[J]
        proj = (lambda v: v - (a_j.dot(v) / asa) * a_j) if asa != 0.0 else (lambda v: v)
        pq = qjj - (np.outer(a_j, a_j @ qjj) / asa if asa != 0.0 else 0.0)
        pqp = pq - (np.outer(pq @ a_j, a_j) / asa if asa != 0.0 else 0.0)
        m = sigma * pqp
        m[np.diag_indices_from(m)] += 1.0
        y = scipy.linalg.cho_solve(scipy.linalg.cho_factor(m, lower=True), proj(g_j))
        t = -r + sigma * np.asarray(xj.T @ proj(y)).ravel()
    else:
        def gram_p(v):  # X_J^T P X_J v
            z = np.asarray(xj @ v).ravel()
            if asa != 0.0:
                z = z - (a_j.dot(z) / asa) * a_j
            return np.asarray(xj.T @ z).ravel()

        sq = xj.multiply(xj) if hasattr(xj, "multiply") else xj * xj
        colsq = np.asarray(sq.sum(axis=0)).ravel()
        diag = 1.0 + sigma * np.maximum(colsq - (m1 * m1 / asa if asa != 0.0 else 0.0), 0.0)
        target = 0.1 * min(opts.eta, opts.cg_eta_cap,
                           float(np.linalg.norm(grad)) ** (1.0 + opts.tau))

        def done(v):  # Newton residual of the direction built from v
            res = -r - (v + sigma * gram_p(v))
            return float(np.linalg.norm(op.x(sigma * gram_p(res)))) <= target

        t, _ = _pcg(lambda v: v + sigma * gram_p(v), -r, 1.0 / diag, done,
                    16 * opts.cg_max_iters)
    q_dir = op.x(t)
    direction = -s - sigma * hs_apply(free, a, q_dir)
    return direction, q_dir, float(t.dot(t))


def bregman(xt, lam_t, px, lam, u_t, a):
    """B_h between a trial projection (xt, lam_t) at u_t and the base projection
    (px, lam) (csrc/proj.cu bregman_term)."""
    return float(((xt - px) * (u_t - 0.5 * (xt + px) - 0.5 * (lam_t + lam) * a)).sum())


def line_search(w, qw, direction, q_dir, dqd, grad, psi0, u, x_k, sigma, bl, opts, base=None):
    """Armijo backtracking, one projection per trial; ref solver.py:292-319.

    Returns (alpha, w_new, qw_new, psi_new, u_new, (px, lam, free))."""
    gd = float(grad.dot(direction))
    if gd >= 0.0:
        raise LineSearchFailed(f"not a descent direction (g'd = {gd:.3e})")
    x_sq = float(x_k.dot(x_k))
    w_qw = float(w.dot(qw))
    w_qdir = float(w.dot(q_dir))
    alpha = 1.0
    for _ in range(61):
        u_t = u - (sigma * alpha) * q_dir
        pr = project(u_t, bl)
        quad = w_qw + 2.0 * alpha * w_qdir + alpha * alpha * dqd
        if PSI_MODE["mode"] == "delta":
            dpsi = alpha * gd + 0.5 * alpha * alpha * dqd + bregman(
                pr[0], pr[1], base[0], base[1], u_t, bl.a) / sigma
            psi_t = psi0 + dpsi
            ok = dpsi <= opts.mu * alpha * gd
        else:
            psi_t = psi_value(quad, u_t, pr[0], x_sq, sigma)
            ok = psi_t <= psi0 + opts.mu * alpha * gd
        if ok:
            return alpha, w + alpha * direction, qw + alpha * q_dir, psi_t, u_t, pr
        alpha *= opts.backtrack
    raise LineSearchFailed("Armijo backtracking exceeded 60 halvings")


def ssn_solve(st, op, c, bl, alm, ssn, eps_k, delta_k, trace=None):
    """Inner semismooth Newton loop, criteria (A')/(B'); ref solver.py:331-411.

    ``st`` is a dict with keys x, w, qw, sigma, inner_total (mutated)."""
    sigma = st["sigma"]
    coeff = math.sqrt(alm.lambda_min_surrogate / sigma)
    floor = 1e-12 * (1.0 + float(np.linalg.norm(c)))
    x_k = st["x"]
    x_sq = float(x_k.dot(x_k))
    u = x_k - sigma * (st["qw"] + c)
    pr = project(u, bl)
    s = st["w"] - pr[0]
    grad = op.matvec(s)
    its = 0
    converged = False
    exhausted = True
    for _ in range(ssn.max_inner):
        gnorm = float(np.linalg.norm(grad))
        if trace is not None:
            trace.append(gnorm)
        if gnorm <= coeff * eps_k and gnorm <= coeff * delta_k * float(np.linalg.norm(pr[0] - x_k)):
            converged, exhausted = True, False
            break
        if gnorm <= floor:
            converged, exhausted = True, False
            break
        nd = newton_direction_factor if ssn.newton == "factor" else newton_direction
        direction, q_dir, dqd = nd(s, grad, pr[2], sigma, op, bl.a, ssn)
        steepest = False
        if float(grad.dot(direction)) >= 0.0:
            direction = -grad
            q_dir = op.matvec(direction)
            dqd = float(direction.dot(q_dir))
            steepest = True
        psi0 = psi_value(float(st["w"].dot(st["qw"])), u, pr[0], x_sq, sigma)
        delta = PSI_MODE["mode"] == "delta"
        if not delta and ssn.mu * abs(float(grad.dot(direction))) <= 1e-16 * (1.0 + abs(psi0)):
            converged, exhausted = True, False
            break
        try:
            _, st["w"], st["qw"], _, u, pr = line_search(
                st["w"], st["qw"], direction, q_dir, dqd, grad, psi0, u, x_k, sigma, bl, ssn,
                base=pr)
        except LineSearchFailed:
            if steepest:
                exhausted = False
                break
            direction = -grad
            q_dir = op.matvec(direction)
            dqd = float(direction.dot(q_dir))
            if not delta and ssn.mu * float(grad.dot(grad)) <= 1e-16 * (1.0 + abs(psi0)):
                exhausted = False
                break
            try:
                _, st["w"], st["qw"], _, u, pr = line_search(
                    st["w"], st["qw"], direction, q_dir, dqd, grad, psi0, u, x_k, sigma, bl, ssn,
                base=pr)
            except LineSearchFailed:
                exhausted = False
                break
        its += 1
        s = st["w"] - pr[0]
        grad = op.matvec(s)
    if exhausted and trace is not None:
        trace.append(float(np.linalg.norm(grad)))
    st["inner_total"] += its
    return {"u": u, "proj": pr, "iterations": its, "converged": converged,
            "hit_max_inner": exhausted}


def kkt_full(x, op, c, bl):
    """R_KKT = ||x - Pi(x - Qx - c)|| / (1 + ||x||); ref solver.py:414-426."""
    qx = op.matvec(x)
    pr = project(x - qx - c, bl)
    return float(np.linalg.norm(x - pr[0])) / (1.0 + float(np.linalg.norm(x))), pr, qx


def kkt_residual(x, op, c, bl):
    return kkt_full(np.asarray(x, dtype=np.float64), op, c, bl)[0]


def alm_solve(op, c, bl, alm=None, ssn=None, x0=None, w0=None, callback=None):
    """Algorithm 1 outer loop with best-iterate safeguard; ref solver.py:429-530."""
    alm = alm or AlmOpts()
    ssn = ssn or SsnOpts()
    t0 = time.perf_counter()
    n = bl.n
    c = np.asarray(c, dtype=np.float64)
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    w = np.zeros(n) if w0 is None else np.array(w0, dtype=np.float64)
    qw = np.zeros(n) if w0 is None else op.matvec(w)
    st = {"x": x, "w": w, "qw": qw, "sigma": alm.sigma0, "inner_total": 0}
    notes = []
    converged = False
    inner_last = 0
    p_last = None
    res = math.inf
    qx_last = None
    outer = 0
    best = None
    stalled = 0
    for k in range(alm.max_outer + 1):
        res, kpr, qx_last = kkt_full(st["x"], op, c, bl)
        if p_last is None:
            p_last = int(np.count_nonzero(kpr[2]))
        if callback is not None:
            callback(k, res, st["sigma"], p_last, inner_last)
        if best is None or res < best[0]:
            best = (res, st["x"], p_last, objective(op, c, st["x"], qx_last))
            stalled = 0
        elif st["sigma"] >= alm.sigma_max:
            stalled += 1
            if stalled >= 3:
                notes.append("stagnated at the attainable accuracy for sigma_max; "
                             "returning the best iterate")
                break
        if res < alm.tol_kkt:
            converged = True
            break
        if k == alm.max_outer:
            notes.append(f"max_outer={alm.max_outer} reached")
            break
        st["qw"] = op.matvec(st["w"])
        inner = ssn_solve(st, op, c, bl, alm, ssn, alm.eps_seq(k), alm.delta_seq(k))
        if inner["hit_max_inner"]:
            notes.append(f"inner solver hit max_inner at outer iteration {k}")
        st["x"] = inner["proj"][0]
        p_last = int(np.count_nonzero(inner["proj"][2]))
        inner_last = inner["iterations"]
        st["sigma"] = min(st["sigma"] * alm.sigma_growth, alm.sigma_max)
        outer += 1
    if best is not None and best[0] < res:
        res, x_ret, p_ret, obj = best
    else:
        x_ret, p_ret = st["x"], p_last
        obj = objective(op, c, st["x"], qx_last)
    return {
        "x_opt": x_ret, "kkt_residual": res, "outer_iters": outer,
        "avg_inner_iters": st["inner_total"] / max(outer, 1),
        "total_inner_iters": st["inner_total"], "unbounded_support_count": int(p_ret),
        "objective": obj, "wall_time": time.perf_counter() - t0,
        "converged": converged, "warnings": notes,
    }
