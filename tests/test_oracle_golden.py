"""Pin the numpy oracle to vectors produced by the real reference package."""

import numpy as np
import pytest

import oracle as O
from conftest import load_cases


def _bl(c):
    return O.BoxLine(c["a"], c["d"], c["l"], c["u"])


def test_projection_matches_reference():
    for c in load_cases("projection.npz", "p"):
        bl = _bl(c)
        x, lam, free = O.project(c["v"], bl)
        scale = 1.0 + np.abs(c["x"]).max()
        assert np.abs(x - c["x"]).max() <= 1e-12 * scale
        assert abs(lam - c["lam"]) <= 1e-12 * (1.0 + abs(c["lam"]))
        np.testing.assert_array_equal(free.astype(np.uint8), c["free"])
        np.testing.assert_array_equal(O.breakpoints(c["v"], bl), c["bp"])
        assert O.grad_phi(0.0, c["v"], bl) == pytest.approx(c["gphi0"], rel=1e-12, abs=1e-12)


def test_hs_jacobian_matches_reference():
    for c in load_cases("hs_jacobian.npz", "h"):
        py = O.hs_apply(c["free"].astype(bool), c["a"], c["y"])
        np.testing.assert_allclose(py, c["py"], rtol=0, atol=1e-13)


def test_newton_direction_matches_reference():
    for c in load_cases("newton.npz", "n"):
        q = c["G"].T @ c["G"]
        op = O.DenseQ(q)
        bl = _bl(c)
        sigma = c["sigma"]
        u = c["x"] - sigma * (q @ c["w"] + c["c"])
        x, lam, free = O.project(u, bl)
        np.testing.assert_array_equal(free.astype(np.uint8), c["free"])
        s = c["w"] - x
        d, qd, dqd = O.newton_direction(s, q @ s, free, sigma, op, bl.a, O.SsnOpts())
        sc = 1.0 + np.linalg.norm(c["qdir"])
        assert np.linalg.norm(qd - c["qdir"]) <= 1e-9 * sc
        assert abs(dqd - c["dqd"]) <= 1e-9 * (1.0 + abs(c["dqd"]))


def test_kkt_residual_matches_reference():
    for c in load_cases("kkt.npz", "k"):
        op = O.DenseQ(c["G"].T @ c["G"])
        r = O.kkt_residual(c["x"], op, c["c"], _bl(c))
        assert r == pytest.approx(c["kkt"], rel=1e-12)


def _problem(c):
    if c["kind"] == "dense":
        return O.DenseQ(c["G"].T @ c["G"]), c["c"], _bl(c)
    if c["kind"] == "csvc":
        return O.csvc_problem(c["A"], c["y"], c["C"])
    return O.svr_problem(c["A"], c["t"], c["C"], c["eps"])


def test_alm_solve_matches_reference():
    for c in load_cases("solve.npz", "s"):
        op, cc, bl = _problem(c)
        rep = O.alm_solve(op, cc, bl, O.AlmOpts(tol_kkt=c["tol"]))
        assert rep["converged"] == bool(c["converged"])
        if c["converged"]:
            assert rep["kkt_residual"] < c["tol"]
        assert rep["objective"] == pytest.approx(c["obj"], rel=1e-6, abs=1e-9)
        if c["kind"] == "dense":  # same operator arithmetic => same iterates, bit for bit
            assert rep["kkt_residual"] == c["kkt"]
            assert (rep["outer_iters"], rep["total_inner_iters"]) == (c["outer"], c["inner"])
        x_ref = c["x_opt"]
        assert np.linalg.norm(rep["x_opt"] - x_ref) <= 1e-4 * (1 + np.linalg.norm(x_ref))


def test_alm_solve_delta_mode_matches_reference_counts():
    """The delta line search (Armijo on psi differences) takes the
    reference's steps on every golden SVM case: same outer/inner counts and solution."""
    O.set_psi_mode("delta")
    try:
        for c in load_cases("solve.npz", "s"):
            if c["kind"] == "dense":
                continue
            op, cc, bl = _problem(c)
            rep = O.alm_solve(op, cc, bl, O.AlmOpts(tol_kkt=c["tol"]))
            assert rep["converged"] and rep["kkt_residual"] < c["tol"]
            assert (rep["outer_iters"], rep["total_inner_iters"]) == (c["outer"], c["inner"])
            assert rep["objective"] == pytest.approx(c["obj"], rel=1e-6, abs=1e-9)
    finally:
        O.set_psi_mode("reference")


def test_bregman_term_is_the_psi_difference():
    """psi(w + a d) - psi(w) = a g'd + a^2 d'Qd / 2 + B_h / sigma exactly (up to
    rounding) for random dense data: the identity the delta mode rests on."""
    rng = np.random.default_rng(7)
    n, q = 300, 20
    A = rng.standard_normal((n, q))
    y = np.where(rng.standard_normal(n) > 0, 1.0, -1.0)
    op, c, bl = O.csvc_problem(A, y, 1.0)
    x = np.clip(rng.random(n), 0, 1.0)
    w = rng.standard_normal(n) * 0.1
    d = rng.standard_normal(n) * 0.1
    sigma = 3.0
    qw, qd = op.matvec(w), op.matvec(d)
    u = x - sigma * (qw + c)
    px, lam, _ = O.project(u, bl)
    O.set_psi_mode("stable")
    try:
        psi0 = O.psi_value(float(w @ qw), u, px, float(x @ x), sigma)
        gd = float((w - px) @ qd)
        for alpha in (1.0, 0.5, 1e-3):
            ut = u - sigma * alpha * qd
            pt, lt, _ = O.project(ut, bl)
            wt = w + alpha * d
            psi_t = O.psi_value(float(wt @ op.matvec(wt)), ut, pt, float(x @ x), sigma)
            dpsi = alpha * gd + 0.5 * alpha ** 2 * float(d @ qd) + O.bregman(pt, lt, px, lam, ut,
                                                                              bl.a) / sigma
            assert dpsi == pytest.approx(psi_t - psi0, rel=1e-9, abs=1e-12)
    finally:
        O.set_psi_mode("reference")


def _factor_ops(c):
    """The golden case's Q = G'G as a dense and a CSR factor X = G' (n x k)."""
    import scipy.sparse as sp

    X = np.ascontiguousarray(c["G"].T)
    Xs = sp.csr_matrix(X)
    return [O.FactoredQ(X), O.CsrFactoredQ(Xs.indptr, Xs.indices, Xs.data, X.shape)]


def test_factor_newton_direction_matches_reference():
    """newton_direction_factor (the oracle route for configs 2-4 at full size) gives the
    reference's Qd, d'Qd and d on every golden Newton case, on all three routes
    (q x q Cholesky, p x p Woodbury, Jacobi-PCG) and for dense and CSR factors."""
    checked = {"q": 0, "p": 0, "cg": 0}
    for c in load_cases("newton.npz", "n"):
        q = c["G"].T @ c["G"]
        bl = _bl(c)
        sigma = c["sigma"]
        u = c["x"] - sigma * (q @ c["w"] + c["c"])
        x, lam, free = O.project(u, bl)
        s = c["w"] - x
        p, k = int(free.sum()), c["G"].shape[0]
        routes = {"q": O.SsnOpts(direct_solve_threshold=max(k, 1)),
                  "cg": O.SsnOpts(direct_solve_threshold=0, cg_eta_cap=1e-15)}
        if 0 < p < k:
            routes["p"] = O.SsnOpts(direct_solve_threshold=p)
        for op in _factor_ops(c):
            for name, opts in routes.items():
                d, qd, dqd = O.newton_direction_factor(s, op.matvec(s), free, sigma, op, bl.a,
                                                       opts)
                tol = 1e-9 if name != "cg" else 1e-7
                sc = 1.0 + np.linalg.norm(c["qdir"])
                assert np.linalg.norm(qd - c["qdir"]) <= tol * sc, (name, p, k)
                assert abs(dqd - c["dqd"]) <= tol * (1.0 + abs(c["dqd"])), (name, p, k)
                assert np.linalg.norm(d - c["dir"]) <= tol * (1.0 + np.linalg.norm(c["dir"]))
                checked[name] += 1
    assert all(v > 0 for v in checked.values()), checked


@pytest.mark.parametrize("mode", ["reference", "delta"])
def test_factor_route_solves_golden_svm_cases(mode):
    """alm_solve with the factor-space Newton route (dense and CSR samples) reproduces
    the reference's outer/inner counts and objective on the golden SVM cases."""
    import scipy.sparse as sp

    O.set_psi_mode(mode)
    try:
        for c in load_cases("solve.npz", "s"):
            if c["kind"] == "dense":
                continue
            probs = [_problem(c)]
            if c["kind"] == "csvc":
                A = sp.csr_matrix(c["A"])
                probs.append(O.csvc_problem_csr(A.indptr, A.indices, A.data, A.shape, c["y"],
                                                c["C"]))
            for op, cc, bl in probs:
                rep = O.alm_solve(op, cc, bl, O.AlmOpts(tol_kkt=c["tol"]),
                                  O.SsnOpts(newton="factor"))
                assert rep["converged"] and rep["kkt_residual"] < c["tol"]
                assert (rep["outer_iters"], rep["total_inner_iters"]) == (c["outer"], c["inner"])
                assert rep["objective"] == pytest.approx(c["obj"], rel=1e-8, abs=1e-9)
    finally:
        O.set_psi_mode("reference")
