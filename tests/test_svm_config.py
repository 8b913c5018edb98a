"""SvmConfig validation and the reference-shaped builders' argument handling (CPU: no
device work; ref svm.py:42-63, 95-127)."""

import pytest

from paper_1910_01312_b200 import errors


def test_svm_config_validation_matches_reference():
    from paper_1910_01312_b200.svm import KernelSpec, SvmConfig

    SvmConfig()
    SvmConfig(task="regression", C=2.0, epsilon=0.1)
    for kw in ({"task": "ranking"}, {"C": 0.0}, {"C": -1.0}, {"epsilon": -0.1},
               {"approx": "sketch"}, {"approx": "nystrom", "approx_size": 0}):
        with pytest.raises(errors.InputError):
            SvmConfig(**kw)
    with pytest.raises(errors.InputError):
        KernelSpec(kind="poly")
    with pytest.raises(errors.InputError):
        KernelSpec(kind="rbf", alpha=0.0)


def test_out_of_scope_kernels_are_rejected_loudly():
    from paper_1910_01312_b200.svm import KernelSpec, SvmConfig, _config_and_c

    with pytest.raises(errors.InputError):
        _config_and_c(SvmConfig(kernel=KernelSpec(kind="rbf", alpha=1.0)))
    with pytest.raises(errors.InputError):
        _config_and_c(SvmConfig(approx="rff", approx_size=10))
    cfg = _config_and_c(2.5, 0.3, "regression")
    assert (cfg.C, cfg.epsilon, cfg.task) == (2.5, 0.3, "regression")


def test_box_line_set_scalar_bounds_match_vector_bounds():
    """Scalar l / u (the SVM builders' constant box) give the same feasibility range and
    errors as the reference's vector form (ref projection.py:29-54)."""
    import numpy as np

    from paper_1910_01312_b200.projection import BoxLineSet

    class _NoDevice:
        device = None

    rng = np.random.default_rng(4)
    n = 1000
    a = np.where(rng.random(n) < 0.3, 1.0, -1.0) * rng.choice([1.0, 2.5], n)
    for l, u in ((0.0, 1.0), (-0.5, 3.0)):
        s = BoxLineSet(a, 0.7, l, u, backend=_NoDevice(), a_device=object())
        v = BoxLineSet(a, 0.7, np.full(n, l), np.full(n, u), backend=_NoDevice(), a_device=object())
        assert s._range_lo == pytest.approx(v._range_lo, rel=1e-14)
        assert s._range_hi == pytest.approx(v._range_hi, rel=1e-14)
        assert (s.l_const, s.u_const, s.l_dev, s.u_dev) == (l, u, None, None)
    with pytest.raises(errors.InfeasibleProblemError):
        BoxLineSet(np.ones(n), n + 1.0, 0.0, 1.0, backend=_NoDevice(), a_device=object())
    with pytest.raises(errors.InputError):
        BoxLineSet(np.ones(n), 0.0, 1.0, 1.0, backend=_NoDevice(), a_device=object())
