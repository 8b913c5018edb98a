"""B200-native (sm_100a) SSsNAL hot path for the unified SVM dual QP.

    min 1/2 x'Qx + c'x   s.t.   a'x = d,  l <= x <= u,   Q = X X^T

A drop-in for the solver path of the reference package ``ssnal`` (arXiv
1910.01312): same entry points, arguments, report fields and errors, with
every arithmetic step of the semismooth-Newton ALM loop running in the
hand-written CUDA library ``_ssnal_b200.so`` (C-ABI: include/ssnal_b200.h).
There is no CPU fallback.
"""

from .errors import (
    CudaUnavailableError,
    InfeasibleProblemError,
    InputError,
    InternalError,
    LineSearchError,
    SsnalError,
)

__version__ = "0.1.0"

_LAZY = {
    "BoxLineSet": "projection", "ActiveSetMask": "projection", "ProjectionResult": "projection",
    "project_box_line": "projection", "hs_jacobian_apply": "projection",
    "LinearKernelOperator": "operators", "DenseOperator": "operators",
    "AlmOptions": "solver", "SsnOptions": "solver", "SolverState": "solver",
    "SolveReport": "solver", "QpProblem": "solver", "alm_solve": "solver",
    "ssn_solve": "solver", "kkt_residual": "solver",
    "build_csvc_dual": "svm", "build_svr_dual": "svm", "recover_bias": "svm",
    "primal_weights": "svm", "SvmConfig": "svm", "SvmModel": "svm", "KernelSpec": "svm",
    "train": "svm", "decision_function": "svm", "predict": "svm", "evaluate": "svm",
    "grad_phi": "api", "breakpoints": "api", "psi_eval": "api", "psi_grad": "api",
    "newton_direction": "api", "line_search": "api",
    "CsrKernelOperator": "operators",
    "CudaBackend": "backend", "default_backend": "backend",
}


def __getattr__(name):
    # torch-importing submodules load on first use so `import paper_1910_01312_b200`
    # (e.g. for datagen) stays light.
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib

    return getattr(importlib.import_module(f".{mod}", __name__), name)


__all__ = sorted(list(_LAZY) + ["CudaUnavailableError", "InfeasibleProblemError", "InputError",
                                "InternalError", "LineSearchError", "SsnalError"])
