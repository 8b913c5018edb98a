"""Host-side solver logic on the CPU (no GPU): the device control flow of
solver._Engine driven by the TEST-ONLY CpuTestBackend, checked against golden
reference runs.  Verifies the factor-space Newton system reproduces the
reference's iterates (same outer/inner counts on the SVM duals)."""

import numpy as np
import pytest
import torch

from conftest import load_cases
from cpu_backend import CpuTestBackend


@pytest.fixture(scope="module")
def mods():
    from paper_1910_01312_b200 import operators, projection, solver, svm

    return operators, projection, solver, svm


def _problem(mods, c, be):
    operators, projection, solver, svm = mods
    if c["kind"] == "dense":
        return solver.QpProblem(operators.DenseOperator(c["G"].T @ c["G"], backend=be), c["c"],
                                projection.BoxLineSet(c["a"], c["d"], c["l"], c["u"], backend=be))
    if c["kind"] == "csvc":
        return svm.build_csvc_dual(c["A"], c["y"], c["C"], backend=be)
    return svm.build_svr_dual(c["A"], c["t"], c["C"], c["eps"], backend=be)


@pytest.mark.parametrize("psi_eval", ["stable", "delta"])
def test_alm_solve_host_logic_matches_reference(mods, psi_eval):
    solver = mods[2]
    be = CpuTestBackend()
    for c in load_cases("solve.npz", "s"):
        rep = solver.alm_solve(_problem(mods, c, be), solver.AlmOptions(tol_kkt=c["tol"]),
                               solver.SsnOptions(psi_eval=psi_eval))
        assert rep.objective == pytest.approx(c["obj"], rel=1e-6, abs=1e-9)
        if c["kind"] != "dense":
            assert rep.converged and rep.kkt_residual < c["tol"]
            assert (rep.outer_iters, rep.total_inner_iters) == (c["outer"], c["inner"])
            np.testing.assert_allclose(rep.x_opt, c["x_opt"], atol=1e-8)


def test_newton_direction_factor_space_matches_reference(mods):
    operators, projection, solver, _ = mods
    be = CpuTestBackend()
    for c in load_cases("newton.npz", "n"):
        q = c["G"].T @ c["G"]
        pb = solver.QpProblem(operators.DenseOperator(q, backend=be), c["c"],
                              projection.BoxLineSet(c["a"], c["d"], c["l"], c["u"], backend=be))
        eng = pb.engine()
        sc, cur = eng.start_inner(torch.from_numpy(c["x"]), torch.from_numpy(c["w"].copy()),
                                  torch.from_numpy(q @ c["w"]), c["sigma"])
        np.testing.assert_array_equal(eng.free.numpy(), c["free"])
        eng.direction(int(cur["nfree"]), c["sigma"], float(cur["sum_a2_free"]))
        sc, _ = eng.fetch(info=True)
        assert np.linalg.norm(eng.qdir.numpy() - c["qdir"]) <= 1e-10 * (1 + np.linalg.norm(c["qdir"]))
        assert sc[3] == pytest.approx(c["dqd"], rel=1e-9, abs=1e-12)


def test_batched_line_search_picks_reference_alpha(mods):
    """Armijo with batched step lengths returns the same alpha as sequential halving."""
    operators, projection, solver, svm = mods
    be = CpuTestBackend()
    c = load_cases("solve.npz", "s")[12]  # config 0
    for batch in (1, 3, 4):
        pb = svm.build_csvc_dual(c["A"], c["y"], c["C"], backend=be)
        rep = solver.alm_solve(pb, solver.AlmOptions(tol_kkt=c["tol"]),
                               solver.SsnOptions(line_search_batch=batch))
        assert (rep.outer_iters, rep.total_inner_iters) == (c["outer"], c["inner"])


def test_workload_solve_options_are_reference_options():
    """datagen.solve_options / tuned_alm_options only name fields of the reference-shaped
    AlmOptions / SsnOptions (ref solver.py:73-95) and leave the dense configs on the
    defaults; the oracle's option classes accept the same keywords (bench.py feeds both
    arms from one table)."""
    import dataclasses

    import oracle as O
    from paper_1910_01312_b200 import datagen, solver

    alm_fields = {f.name for f in dataclasses.fields(solver.AlmOptions)}
    ssn_fields = {f.name for f in dataclasses.fields(solver.SsnOptions)}
    sparse = datagen.solve_options({"indptr": None})
    assert set(sparse["alm"]) <= alm_fields and set(sparse["ssn"]) <= ssn_fields
    assert sparse["alm"]["sigma_max"] == 625.0 and sparse["ssn"]["max_inner"] == 200
    O.AlmOpts(tol_kkt=1e-6, **sparse["alm"])
    O.SsnOpts(newton="factor", **sparse["ssn"])
    for cfg in ({"A": None, "task": "csvc"}, {"A": None, "task": "svr"}):
        assert datagen.solve_options(cfg) == {"alm": {}, "ssn": {}}
    assert datagen.tuned_alm_options({"A": None, "task": "csvc"}) is None
    assert datagen.tuned_alm_options({"indptr": None, "task": "csvc"}) is None
    tuned = datagen.tuned_alm_options({"A": None, "task": "svr"})
    assert set(tuned) <= alm_fields
    solver.AlmOptions(tol_kkt=1e-6, **tuned)


def test_bench_cpu_sample_shapes():
    """bench.py's bounded CPU sample of the sparse configs scales n and q of the SAME
    generator (no oracle solve here)."""
    import inspect
    import os
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_1910_01312_b200 import datagen

    for k, div in bench.CPU_SAMPLE_DIV.items():
        sig = inspect.signature(datagen.CONFIGS[k]).parameters
        n, q = sig["n"].default // div, sig["q"].default // div
        assert n >= 10_000 and q >= 1_000
    small = datagen.make_config(3, n=2000, q=500)
    assert small["shape"] == (2000, 500) and small["indptr"][-1] == small["indices"].size
