"""Kernel-level parity of the sm_100a library against the oracle / golden vectors.

Tolerances (BASELINE north_star): projection and operator products within
1e-12 relative, free set J bit-exact given identical input vectors.
"""

import numpy as np
import pytest
import torch

import oracle as O
from conftest import load_cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import __graft_entry__ as g

    g.build()
    import paper_1910_01312_b200 as P

    return P


def _dev(x, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device="cuda")


def test_projection_golden(pkg):
    for c in load_cases("projection.npz", "p"):
        box = pkg.BoxLineSet(c["a"], c["d"], c["l"], c["u"])
        r = pkg.project_box_line(c["v"], box)
        x = r.x.cpu().numpy()
        scale = 1.0 + np.abs(c["x"]).max()
        assert np.abs(x - c["x"]).max() <= 1e-12 * scale, (c["v"].size, np.abs(x - c["x"]).max())
        assert abs(r.lambda_hat - c["lam"]) <= 1e-12 * (1.0 + abs(c["lam"]))
        np.testing.assert_array_equal(r.active_mask.free_mask.cpu().numpy(), c["free"])


def test_projection_random_vs_oracle(pkg):
    rng = np.random.default_rng(11)
    for trial in range(60):
        n = int(rng.choice([1, 7, 100, 1000, 20000, 200000]))
        a = rng.standard_normal(n)
        a[rng.random(n) < 0.1] = 0.0
        if trial % 3 == 0:  # SVM shape
            a = np.where(rng.random(n) < 0.5, 1.0, -1.0)
            l, u = np.zeros(n), np.full(n, float(rng.choice([0.1, 1.0, 64.0])))
        else:
            l, u = -rng.random(n) - 0.1, rng.random(n) + 0.1
        d = float(a @ (l + rng.random(n) * (u - l)))
        v = rng.standard_normal(n) * rng.choice([0.5, 3.0, 100.0])
        if trial % 5 == 0:  # heavy duplication of breakpoints
            v = np.round(v, 1)
        bl = O.BoxLine(a, d, l, u)
        x_ref, lam_ref, free_ref = O.project(v, bl)
        r = pkg.project_box_line(v, pkg.BoxLineSet(a, d, l, u))
        x = r.x.cpu().numpy()
        assert np.abs(x - x_ref).max() <= 1e-12 * (1.0 + np.abs(x_ref).max())
        assert abs(r.lambda_hat - lam_ref) <= 1e-12 * (1.0 + abs(lam_ref))
        np.testing.assert_array_equal(r.active_mask.free_mask.cpu().numpy().astype(bool), free_ref)
        # feasibility at the reference's stated tolerances
        assert abs(a @ x - d) <= 1e-9 * (1.0 + abs(d)) + 1e-12 * np.abs(a).sum() * np.abs(x).max()


@pytest.mark.parametrize("newton,hint_kind", [(0, "zero"), (1, "zero"), (3, "zero"),
                                              (3, "near"), (8, "far"), (2, "near")])
def test_projection_search_modes(pkg, newton, hint_kind):
    """Every root-search route (pure K-ary, Newton then K-ary fallback, warm and cold
    Newton) lands on the reference's multiplier and free set."""
    from paper_1910_01312_b200 import _lib

    rng = np.random.default_rng(100 + newton)
    for trial in range(25):
        n = int(rng.choice([3, 50, 5000, 60000]))
        if trial % 2:
            a = np.where(rng.random(n) < 0.5, 1.0, -1.0)
            l, u = np.zeros(n), np.full(n, 1.0)
        else:
            a = rng.standard_normal(n)
            a[rng.random(n) < 0.1] = 0.0
            l, u = -rng.random(n) - 0.1, rng.random(n) + 0.1
        d = float(a @ (l + rng.random(n) * (u - l)))
        v = rng.standard_normal(n) * rng.choice([0.5, 5.0, 1e3])
        if trial % 5 == 0:
            v = np.round(v, 1)
        bl = O.BoxLine(a, d, l, u)
        x_ref, lam_ref, free_ref = O.project(v, bl)
        box = pkg.BoxLineSet(a, d, l, u)
        be = box.backend
        hint = {"zero": 0.0, "near": lam_ref * (1 + 1e-3) + 1e-6, "far": lam_ref + 1e3}[hint_kind]
        states = be.new_states(1)
        xo = be.empty(n)
        fo = be.empty(n, torch.uint8)
        be.project(_dev(v), box, states, x_out=xo, free_out=fo, hint=hint, newton=newton,
                   passes=2, phases=7 if newton == 0 else 6)
        st = be.read_states(states.cpu())
        rounds = 0
        while st["status"][0] != _lib.PROJ_APPLIED:
            rounds += 1
            assert rounds < 20
            be.project(_dev(v), box, states, x_out=xo, free_out=fo, phases=6, passes=8, newton=0)
            st = be.read_states(states.cpu())
        assert np.abs(xo.cpu().numpy() - x_ref).max() <= 1e-12 * (1.0 + np.abs(x_ref).max())
        assert abs(float(st["lam"][0]) - lam_ref) <= 1e-12 * (1.0 + abs(lam_ref))
        np.testing.assert_array_equal(fo.cpu().numpy().astype(bool), free_ref)


def test_projection_batched_trials(pkg):
    from paper_1910_01312_b200 import backend as B

    rng = np.random.default_rng(3)
    n = 50000
    y = np.where(rng.random(n) < 0.5, 1.0, -1.0)
    box = pkg.BoxLineSet(y, 0.0, np.zeros(n), np.ones(n))
    be = box.backend
    u = rng.standard_normal(n) * 2
    qd = rng.standard_normal(n)
    coefs = [3.0 * 0.5 ** j for j in range(4)]
    states = be.new_states(4)
    xo = be.empty((4, n))
    fo = be.empty((4, n), torch.uint8)
    st = be.project_sync(_dev(u), box, states, T=4, B=_dev(qd), coefs=coefs, x_out=xo, free_out=fo)
    bl = O.BoxLine(y, 0.0, np.zeros(n), np.ones(n))
    for t, cf in enumerate(coefs):
        v = u - cf * qd
        x_ref, lam_ref, free_ref = O.project(v, bl)
        assert np.abs(xo[t].cpu().numpy() - x_ref).max() <= 1e-12
        np.testing.assert_array_equal(fo[t].cpu().numpy().astype(bool), free_ref)
        assert st["sum_v2"][t] == pytest.approx(v @ v, rel=1e-12)
        assert st["sum_r2"][t] == pytest.approx(((v - x_ref) ** 2).sum(), rel=1e-10, abs=1e-14)
        assert st["nfree"][t] == free_ref.sum()
    del B


@pytest.mark.parametrize("T", [1, 2, 3, 5, 8])
def test_projection_batched_trials_large_n(pkg, T):
    """n above the cluster kernel's capacity: the multi-trial cooperative kernel (every
    trial of the batch from ONE read of u, Qd, a per pass) matches the oracle trial by
    trial; eps-SVR-shaped constraint a = (e; -e)."""
    rng = np.random.default_rng(30 + T)
    m = 150_000
    n = 2 * m
    a = np.concatenate([np.ones(m), -np.ones(m)])
    box = pkg.BoxLineSet(a, 0.0, np.zeros(n), np.ones(n))
    be = box.backend
    u = rng.standard_normal(n) * 2
    qd = rng.standard_normal(n)
    coefs = [5.0 * 0.5 ** j for j in range(T)]
    states = be.new_states(T)
    xo = be.empty((T, n))
    fo = be.empty((T, n), torch.uint8)
    st = be.project_sync(_dev(u), box, states, T=T, B=_dev(qd), coefs=coefs, x_out=xo,
                         free_out=fo, hint=0.3)
    bl = O.BoxLine(a, 0.0, np.zeros(n), np.ones(n))
    for t, cf in enumerate(coefs):
        v = u - cf * qd
        x_ref, lam_ref, free_ref = O.project(v, bl)
        assert abs(float(st["lam"][t]) - lam_ref) <= 1e-12 * (1.0 + abs(lam_ref))
        assert np.abs(xo[t].cpu().numpy() - x_ref).max() <= 1e-12
        np.testing.assert_array_equal(fo[t].cpu().numpy().astype(bool), free_ref)
        assert st["sum_v2"][t] == pytest.approx(v @ v, rel=1e-12)
        assert st["sum_r2"][t] == pytest.approx(((v - x_ref) ** 2).sum(), rel=1e-10, abs=1e-14)
        assert st["nfree"][t] == free_ref.sum()


def test_hs_jacobian_golden(pkg):
    for c in load_cases("hs_jacobian.npz", "h"):
        py = pkg.hs_jacobian_apply(_dev(c["free"], torch.uint8), c["a"], c["y"]).cpu().numpy()
        np.testing.assert_allclose(py, c["py"], rtol=0, atol=1e-13)


def test_dots_vec_compact(pkg):
    be = pkg.default_backend()
    rng = np.random.default_rng(5)
    for n in (1, 33, 4097, 1_000_003):
        xs = [rng.standard_normal(n) for _ in range(3)]
        m = (rng.random(n) < 0.3).astype(np.uint8)
        out = be.zeros(8)
        be.dots([(_dev(xs[0]), _dev(xs[1])), (_dev(xs[2]), None)], out, mask=_dev(m, torch.uint8))
        o = out.cpu().numpy()
        mb = m.astype(bool)
        assert o[0] == pytest.approx(float(xs[0][mb] @ xs[1][mb]), rel=1e-12, abs=1e-12)
        assert o[1] == pytest.approx(float(xs[2][mb] @ xs[2][mb]), rel=1e-12, abs=1e-12)
        # vec op 0: x + alpha (y + z), numpy rounding order -> bit exact
        r = be.empty(n)
        be.vec(0, -2.5, _dev(xs[0]), _dev(xs[1]), _dev(xs[2]), r)
        np.testing.assert_array_equal(r.cpu().numpy(), xs[0] + (-2.5) * (xs[1] + xs[2]))
        be.vec(1, 0.0, _dev(xs[0]), _dev(xs[1]), _dev(xs[2]), r)
        np.testing.assert_array_equal(r.cpu().numpy(), (xs[0] - xs[1]) - xs[2])
        idx = be.zeros(n, torch.int32)
        cnt = be.zeros(1, torch.int64)
        be.compact(_dev(m, torch.uint8), idx, cnt)
        p = int(cnt.cpu()[0])
        np.testing.assert_array_equal(idx[:p].cpu().numpy(), np.flatnonzero(m))


@pytest.mark.parametrize("shape,svr,signed", [((1000, 50), False, True), ((3001, 300), False, True),
                                              ((777, 500), True, False), ((20000, 333), False, False),
                                              ((64, 7), True, False)])
def test_dense_products(pkg, shape, svr, signed):
    rng = np.random.default_rng(shape[0])
    n, q = shape
    A = rng.standard_normal((n, q))
    y = np.where(rng.random(n) < 0.5, 1.0, -1.0) if signed else None
    op = pkg.LinearKernelOperator(A, labels=y, svr_block=svr)
    X = (y[:, None] * A) if signed else A
    if svr:
        X = np.vstack([A, -A])
    v1, v2 = rng.standard_normal(X.shape[0]), rng.standard_normal(X.shape[0])
    g = op.xt([_dev(v1), _dev(v2)]).cpu().numpy()
    ref = X.T @ np.stack([v1, v2], axis=1)
    assert np.abs(g.T - ref).max() <= 1e-12 * np.abs(X).sum(axis=0).max() * max(np.abs(v1).max(), 1)
    d = rng.standard_normal((2, q))
    out = op.x(_dev(d), k=2).cpu().numpy()
    ref = X @ d.T
    assert np.abs(out.T - ref).max() <= 1e-12 * np.abs(X).sum(axis=1).max() * np.abs(d).max()


@pytest.mark.parametrize("m", [1, 7, 33, 115, 160, 161, 300, 500, 517, 768, 769, 1100, 2048])
def test_cholesky_solve_sizes(pkg, m):
    """Every Cholesky route: shared-memory resident (m <= 160), grid-wide cooperative with
    inverted diagonal blocks (m <= 2048)."""
    be = pkg.default_backend()
    rng = np.random.default_rng(m)
    G = rng.standard_normal((m, m + 3))
    M = np.eye(m) + 3.0 * G @ G.T
    b = rng.standard_normal(m)
    Md = _dev(M)
    xo = be.empty(m)
    info = be.zeros(1, torch.int32)
    be.chol_solve(Md, m, _dev(b), -2.0, xo, info)
    assert int(info.cpu()[0]) == 0
    x_ref = -2.0 * np.linalg.solve(M, b)
    assert np.linalg.norm(xo.cpu().numpy() - x_ref) <= 1e-12 * np.linalg.cond(M) * np.linalg.norm(x_ref)
    # not SPD -> info reports the failing column
    Mbad = M.copy()
    Mbad[m // 2, m // 2] = -1.0
    be.chol_solve(_dev(Mbad), m, _dev(b), 1.0, xo, info)
    assert int(info.cpu()[0]) > 0


@pytest.mark.parametrize("n,q,p", [(500, 50, 37), (5000, 300, 300), (3000, 130, 1), (9000, 500, 2000)])
def test_gram_and_cholesky(pkg, n, q, p):
    rng = np.random.default_rng(q)
    A = rng.standard_normal((n, q))
    y = np.where(rng.random(n) < 0.5, 1.0, -1.0)
    op = pkg.LinearKernelOperator(A, labels=y)
    be = op.backend
    J = np.sort(rng.choice(n, size=p, replace=False)).astype(np.int32)
    Jd = be.zeros(n, torch.int32)
    Jd[:p] = _dev(J, torch.int32)
    pdev = _dev(np.array([p]), torch.int64)
    asa = float(p)  # a = y, a_J'a_J = p
    asa_dev = _dev(np.array([asa]))
    sigma = 7.5
    M = be.empty((q, q))
    m1 = be.empty(q)
    be.dense_gram(op, Jd, pdev, n, _dev(y), sigma, asa_dev, M, m1)
    X = y[:, None] * A
    Z = X[J]
    m1_ref = Z.T @ y[J]
    M_ref = np.eye(q) + sigma * (Z.T @ Z - np.outer(m1_ref, m1_ref) / asa)
    np.testing.assert_allclose(m1.cpu().numpy(), m1_ref, rtol=1e-12, atol=1e-10)
    np.testing.assert_allclose(M.cpu().numpy(), M_ref, rtol=1e-12, atol=1e-9 * sigma * p)
    b = rng.standard_normal(q)
    xo = be.empty(q)
    info = be.zeros(1, torch.int32)
    be.chol_solve(M, q, _dev(b), -1.0, xo, info)
    assert int(info.cpu()[0]) == 0
    x_ref = -np.linalg.solve(M_ref, b)
    assert np.linalg.norm(xo.cpu().numpy() - x_ref) <= 1e-10 * np.linalg.cond(M_ref) * np.linalg.norm(x_ref)


@pytest.mark.parametrize("n,q,nnz_row,zipf", [(3000, 500, 7, False), (20000, 3000, 30, True),
                                              (5, 4, 2, False)])
def test_csr_products(pkg, n, q, nnz_row, zipf):
    """CSR X d and CSC X^T v (segmented, split hot columns) against scipy."""
    import scipy.sparse as sp

    from paper_1910_01312_b200.operators import CsrKernelOperator

    rng = np.random.default_rng(n)
    rows = np.repeat(np.arange(n), nnz_row)
    if zipf:  # a few very hot columns force split segments + folds
        cols = np.minimum(rng.zipf(1.3, size=n * nnz_row) - 1, q - 1)
    else:
        cols = rng.integers(0, q, size=n * nnz_row)
    A = sp.csr_matrix((rng.standard_normal(rows.size), (rows, cols)), shape=(n, q))
    A.sum_duplicates()
    y = np.where(rng.random(n) < 0.5, 1.0, -1.0)
    op = CsrKernelOperator(A, labels=y)
    X = sp.diags(y) @ A
    d = rng.standard_normal(q)
    v = rng.standard_normal(n)
    out = op.x(_dev(d).view(1, -1))[0].cpu().numpy()
    np.testing.assert_allclose(out, X @ d, rtol=1e-12, atol=1e-12 * np.abs(X).sum(axis=1).max())
    g = op.xt([_dev(v)])[0].cpu().numpy()
    np.testing.assert_allclose(g, X.T @ v, rtol=1e-12, atol=1e-11 * max(1, np.abs(X).sum(axis=0).max()))
    if zipf and n > 1000:
        assert op.nslots > 0  # hot columns were split


@pytest.mark.parametrize("keep_frac", [0.0, 0.004, 0.16, 0.7, 1.0])
def test_csr_restricted_products(pkg, keep_frac):
    """X_J^T w on the J-restricted CSC (nnz-balanced chunked segmented sums, chunk-
    crossing segments fixed up in order, split hot columns folded) and X_J d over a
    row list, against scipy.  One column sits in every row (20,000 entries: ten
    2048-entry segments, each spanning several 256-entry chunks); Zipf columns give
    long runs of 0-3-entry segments; J from empty to all rows."""
    import ctypes

    import scipy.sparse as sp

    from paper_1910_01312_b200 import _lib
    from paper_1910_01312_b200.operators import CsrKernelOperator

    rng = np.random.default_rng(int(keep_frac * 1000) + 7)
    n, q, k = 20000, 5000, 12
    rows = np.repeat(np.arange(n), k)
    cols = np.minimum(rng.zipf(1.1, size=n * k) - 1, q - 1)
    cols[::k] = 17  # the all-rows column
    A = sp.csr_matrix((rng.standard_normal(rows.size), (rows, cols)), shape=(n, q))
    A.sum_duplicates()
    y = np.where(rng.random(n) < 0.5, 1.0, -1.0)
    op = CsrKernelOperator(A, labels=y)
    X = (sp.diags(y) @ A).tocsr()
    keep = (rng.random(n) < keep_frac).astype(np.uint8)
    J = np.flatnonzero(keep).astype(np.int32)
    p = J.size
    w = rng.standard_normal(max(p, 1))
    be = pkg.default_backend()
    ws = be.zeros(int(_lib.load().ssnal_csr_restricted_ws_bytes(op._cref)), torch.uint8)
    out = be.empty(q)
    keep_d, J_d, w_d = _dev(keep, torch.uint8), _dev(np.r_[J, 0].astype(np.int32), torch.int32), _dev(w)
    for _ in range(2):  # the second call reuses the workspace (stale entries past nnz_J)
        _lib.call("ssnal_csr_xt_restricted", op._cref, keep_d.data_ptr(), J_d.data_ptr(), p,
                  w_d.data_ptr(), out.data_ptr(), ws.data_ptr(), be.stream())
        ref = X[J].T @ w[:p] if p else np.zeros(q)
        scale = 1e-12 * (float((abs(X[J]).T @ np.abs(w[:p])).max()) if p else 1.0)
        np.testing.assert_allclose(out.cpu().numpy(), ref, rtol=1e-12, atol=scale)
        w = rng.standard_normal(max(p, 1))
        w_d = _dev(w)
    d = rng.standard_normal(q)
    zo = be.empty(max(p, 1))
    if p:
        _lib.call("ssnal_csr_xd", op._cref, J_d.data_ptr(), p, _dev(d).data_ptr(), zo.data_ptr(),
                  be.stream())
        np.testing.assert_allclose(zo.cpu().numpy()[:p], X[J] @ d, rtol=1e-12,
                                   atol=1e-12 * np.abs(X).sum(axis=1).max())
        # packed J-restricted CSR (the CG's X_J d): bit-identical to the row-list product
        z2 = be.empty(p)
        _lib.call("ssnal_csr_xd_restricted", op._cref, keep_d.data_ptr(), J_d.data_ptr(), p,
                  _dev(d).data_ptr(), z2.data_ptr(), ws.data_ptr(), be.stream())
        assert torch.equal(z2, zo[:p])


def test_csr_study_knob_kernels():
    """The measured-and-left-off variants of the CG products stay
    correct: SSNAL_CSR_HOT=1 (shared-memory staging of the hot columns' d entries in X_J d,
    bit-identical to the plain kernel) and SSNAL_CSCJ_T=1 (interleaved loads transposed
    through shared memory in X_J^T w).  The knobs are read once per process, so the
    restricted-product tests run again in a child process with both set."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, SSNAL_CSR_HOT="1", SSNAL_CSCJ_T="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(root, "tests", "test_gpu_kernels.py"),
                        "-q", "-x", "-m", "gpu", "-k", "test_csr_restricted_products"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "5 passed" in r.stdout, r.stdout[-1000:]


@pytest.mark.parametrize("shape,svr,aligned", [((3001, 300), False, True), ((2000, 51), False, False),
                                                ((1500, 64), True, True)])
def test_fused_gradient_and_direction_epilogue(pkg, shape, svr, aligned):
    """ssnal_dense_gradient / ssnal_dense_direction_epilogue against the unfused kernels
    (streaming route when q is even and A 16-byte aligned, fallback otherwise)."""
    from paper_1910_01312_b200 import operators

    be = pkg.default_backend()
    rng = np.random.default_rng(shape[0] + shape[1])
    n_phys, q = shape
    A = _dev(rng.standard_normal((n_phys, q)))
    labels = None if svr else np.where(rng.random(n_phys) < 0.5, 1.0, -1.0)
    op = operators.LinearKernelOperator(A, labels=labels, svr_block=svr)
    n = op.n
    w, xp, a = (_dev(rng.standard_normal(n)) for _ in range(3))
    s, grad, g2 = be.empty(n), be.empty(n), be.zeros(4)
    gr = be.empty((1, q))
    be.dense_gradient(op, w, xp, s, gr[0], grad, g2[0:1])
    s_ref = w - xp
    gr_ref = op.xt([s_ref])
    grad_ref = op.x(gr_ref)[0]
    torch.cuda.synchronize()
    assert torch.equal(s, s_ref)
    np.testing.assert_allclose(gr.cpu().numpy(), gr_ref.cpu().numpy(), rtol=1e-13, atol=1e-12)
    np.testing.assert_allclose(grad.cpu().numpy(), grad_ref.cpu().numpy(), rtol=1e-13, atol=1e-11)
    assert float(g2[0]) == pytest.approx(float(grad_ref @ grad_ref), rel=1e-13)
    # direction epilogue from a random t and free mask
    t = _dev(rng.standard_normal(q))
    free = _dev((rng.random(n) < 0.3).astype(np.uint8), torch.uint8)
    fm = free.cpu().numpy().astype(bool)
    av = a.cpu().numpy()
    asa = be.zeros(1)
    asa[0] = float((av[fm] ** 2).sum())
    qw = _dev(rng.standard_normal(n))
    qdir, dirv, dots4 = be.empty(n), be.empty(n), be.zeros(4)
    sigma = 3.7
    be.direction_epilogue(op, t, qdir, free, a, asa, s, sigma, grad, w, qw, dirv, dots4)
    qd_ref = op.x(t.view(1, -1))[0].cpu().numpy()
    coef = float((av[fm] * qd_ref[fm]).sum()) / float(asa[0])
    d_ref = -s.cpu().numpy() - sigma * np.where(fm, qd_ref - coef * av, 0.0)
    torch.cuda.synchronize()
    np.testing.assert_allclose(qdir.cpu().numpy(), qd_ref, rtol=1e-13, atol=1e-11)
    np.testing.assert_allclose(dirv.cpu().numpy(), d_ref, rtol=1e-11, atol=1e-10)
    ref4 = [grad.cpu().numpy() @ d_ref, w.cpu().numpy() @ qw.cpu().numpy(),
            w.cpu().numpy() @ qd_ref, t.cpu().numpy() @ t.cpu().numpy()]
    np.testing.assert_allclose(dots4.cpu().numpy(), ref4, rtol=1e-10)


def test_cluster_projection_matches_grid_kernel(pkg):
    """The cluster route (n <= 65536, every trial count) and the grid-wide fused route
    (larger n) solve the same projections: lambda to 1e-12, free masks identical."""
    from paper_1910_01312_b200 import projection

    be = pkg.default_backend()
    rng = np.random.default_rng(21)
    for n in (1000, 65536, 70000):  # cluster, cluster (limit), grid-wide
        a = np.where(rng.random(n) < 0.5, 1.0, -1.0)
        v = rng.standard_normal(n) * 2.0
        B = rng.standard_normal(n) * 0.05
        box = projection.BoxLineSet(a, 0.0, np.zeros(n), np.ones(n))
        coefs = [2.0 ** -k for k in range(8)]
        st = be.new_states(8)
        xo = be.empty((8, n))
        fo = be.zeros((8, n), torch.uint8)
        be.project(_dev(v), box, st, 8, B=_dev(B), coefs=coefs, x_out=xo, free_out=fo)
        rec = be.read_states(st.cpu())
        bl = O.BoxLine(a, 0.0, np.zeros(n), np.ones(n))
        for k in range(8):
            x_ref, lam_ref, free_ref = O.project(v - coefs[k] * B, bl)
            assert abs(rec[k]["lam"] - lam_ref) <= 1e-12 * (1 + abs(lam_ref))
            np.testing.assert_allclose(xo[k].cpu().numpy(), x_ref, atol=1e-12)
            np.testing.assert_array_equal(fo[k].cpu().numpy().astype(bool), free_ref)
