"""The C-ABI library builds, loads without a GPU and exports every symbol of
include/ssnal_b200.h (no compute calls here)."""

import os
import re

from conftest import ROOT


def test_build_and_exports():
    import __graft_entry__ as g

    g.build()
    from paper_1910_01312_b200 import _lib

    lib = _lib.load()
    header = open(os.path.join(ROOT, "include", "ssnal_b200.h")).read()
    declared = set(re.findall(
        r"^\s*(?:int|size_t|const char\*|unsigned long long)\s+(ssnal_\w+)\(", header, re.M))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.exported_symbols())
    assert lib.ssnal_proj_state_bytes() == _lib.PROJ_STATE_DTYPE.itemsize
    assert b"sm_100a" in lib.ssnal_version()


def test_no_cpu_fallback_without_cuda():
    import torch

    if torch.cuda.is_available():
        return
    import pytest

    from paper_1910_01312_b200 import CudaUnavailableError, default_backend

    with pytest.raises(CudaUnavailableError):
        default_backend()
