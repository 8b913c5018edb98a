"""The reference's functional API and SVM pipeline on the device, against vectors the
REAL reference produced (tests/golden/*.npz, scripts/make_golden.py):
newton_direction vs newton.npz (Qd, d'Qd, d), grad_phi / breakpoints vs projection.npz,
psi_eval / psi_grad / line_search vs the oracle, recover_bias / train / decision_function
/ evaluate vs svm.npz."""

import numpy as np
import pytest
import torch

import oracle as O
from conftest import load_cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import __graft_entry__ as g

    g.build()
    import paper_1910_01312_b200 as P

    return P


def _qp(P, c):
    q = c["G"].T @ c["G"]
    return q, P.QpProblem(P.DenseOperator(q), c["c"], P.BoxLineSet(c["a"], c["d"], c["l"], c["u"]))


def test_newton_direction_matches_reference_goldens(P):
    """ref solver.py:194-289 on every golden Newton case: q_dir, dir'Q dir and the
    direction representative d = -s - sigma P(Qd), through the device factor-space system."""
    for c in load_cases("newton.npz", "n"):
        q, pb = _qp(P, c)
        sigma = c["sigma"]
        u = c["x"] - sigma * (q @ c["w"] + c["c"])
        proj = P.project_box_line(u, pb.constraint)
        np.testing.assert_array_equal(proj.active_mask.free_mask.cpu().numpy(), c["free"])
        s = c["w"] - proj.x.cpu().numpy()
        d, qd, dqd = P.newton_direction(s, q @ s, proj, sigma, pb, P.SsnOptions())
        sc = 1.0 + np.linalg.norm(c["qdir"])
        assert np.linalg.norm(qd.cpu().numpy() - c["qdir"]) <= 1e-9 * sc
        assert abs(dqd - c["dqd"]) <= 1e-9 * (1.0 + abs(c["dqd"]))
        assert np.linalg.norm(d.cpu().numpy() - c["dir"]) <= 1e-9 * (1 + np.linalg.norm(c["dir"]))


def test_grad_phi_and_breakpoints_match_reference(P):
    for c in load_cases("projection.npz", "p")[:60]:
        box = P.BoxLineSet(c["a"], c["d"], c["l"], c["u"])
        assert P.grad_phi(0.0, c["v"], box) == pytest.approx(c["gphi0"], rel=1e-12, abs=1e-12)
        bp = P.breakpoints(c["v"], box).cpu().numpy()
        np.testing.assert_array_equal(bp, c["bp"])


def test_psi_eval_grad_and_line_search_match_oracle(P):
    rng = np.random.default_rng(5)
    n, k = 400, 12
    A = rng.standard_normal((n, k))
    y = np.where(rng.random(n) < 0.5, 1.0, -1.0)
    pb = P.build_csvc_dual(A, y, P.SvmConfig(C=1.0))
    op, c, bl = O.csvc_problem(A, y, 1.0)
    x = np.clip(rng.random(n), 0, 1)
    w = 0.1 * rng.standard_normal(n)
    sigma = 2.0
    qw = op.matvec(w)
    state = P.SolverState(x=torch.as_tensor(x, device="cuda"), w=None, qw=None, sigma=sigma)
    u = x - sigma * (qw + c)
    px, lam, free = O.project(u, bl)
    O.set_psi_mode("stable")
    try:
        psi_ref = O.psi_value(float(w @ qw), u, px, float(x @ x), sigma)
    finally:
        O.set_psi_mode("reference")
    assert P.psi_eval(w, qw, state, pb) == pytest.approx(psi_ref, rel=1e-12)
    grad, proj = P.psi_grad(w, qw, state, pb)
    np.testing.assert_allclose(grad.cpu().numpy(), op.matvec(w - px), rtol=1e-11, atol=1e-11)
    s = w - px
    d, qd, dqd = P.newton_direction(s, op.matvec(s), proj, sigma, pb, P.SsnOptions())
    d_o, qd_o, dqd_o = O.newton_direction(s, op.matvec(s), free, sigma, op, bl.a, O.SsnOpts())
    np.testing.assert_allclose(qd.cpu().numpy(), qd_o, rtol=1e-9, atol=1e-9)
    alpha, w_new, qw_new, psi_new, u_new, pr_new = P.line_search(
        w, qw, d, qd, dqd, op.matvec(s), psi_ref, u, state, pb, P.SsnOptions())
    O.set_psi_mode("stable")
    try:
        a_o, w_o, qw_o, psi_o, u_o, pr_o = O.line_search(w, qw, d_o, qd_o, dqd_o, op.matvec(s),
                                                         psi_ref, u, x, sigma, bl, O.SsnOpts())
    finally:
        O.set_psi_mode("reference")
    assert alpha == a_o
    assert psi_new == pytest.approx(psi_o, rel=1e-10)
    np.testing.assert_allclose(pr_new.x.cpu().numpy(), pr_o[0], atol=1e-10)


def _cfg(P, c):
    task = str(c["task"])
    return P.SvmConfig(task=task, C=float(c["C"]), epsilon=float(c["eps"]))


def test_recover_bias_matches_reference(P):
    """ref svm.py:147-208 at the reference's own dual solutions, free-set mean and
    interval-midpoint branches, C-SVC and eps-SVR."""
    for c in load_cases("svm.npz", "v"):
        b = P.recover_bias(c["dual_x"], c["A"], c["t"], _cfg(P, c))
        assert b == pytest.approx(c["bias"], rel=1e-10, abs=1e-10)


def test_train_decision_evaluate_match_reference(P):
    """ref svm.py:221-295: the trained model (device solve) has the reference's support
    set, bias and decision values to solver tolerance, and the same metric."""
    for c in load_cases("svm.npz", "v"):
        if c["tol"] == 0.0:
            continue
        model, rep = P.train(c["A"], c["t"], _cfg(P, c), alm_opts=P.AlmOptions(tol_kkt=c["tol"]))
        assert rep.converged
        assert model.bias == pytest.approx(c["bias"], rel=1e-5, abs=1e-5)
        np.testing.assert_array_equal(model.support_indices, c["support_indices"])
        np.testing.assert_allclose(P.decision_function(model, c["points"]), c["decision"],
                                   rtol=1e-5, atol=1e-5)
        metric = list(P.evaluate(model, c["A"], c["t"]).values())[0]
        assert metric == pytest.approx(c["metric"], rel=1e-4, abs=1e-4)
