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


def test_pspace_workspace_bounds_every_smaller_system():
    """ssnal_pspace_ws_bytes(p, q) must cover every system order p' <= p: the split-K
    factor of the row Gram grows as p' shrinks (regression: sized at p = q = 400 the
    workspace was 0.8 MB short for p' = 380, whose partial tiles then ran past it)."""
    from paper_1910_01312_b200 import _lib

    lib = _lib.load()

    def need(p, q):  # csrc/newton.cu gram_ksplit + launch_pspace_direction layout
        nt = -(-p // 64)
        pairs = nt * (nt + 1) // 2
        s = max(1, min(-(-296 // pairs), -(-q // 32), 16))
        return ((s + 1) * p * p + 4 * p + 16 * q + 64) * 8

    for q in (50, 300, 400, 1000, 2048):
        have = lib.ssnal_pspace_ws_bytes(q, q)
        assert all(have >= need(p, q) for p in range(1, q + 1)), q
