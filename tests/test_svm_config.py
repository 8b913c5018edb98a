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
