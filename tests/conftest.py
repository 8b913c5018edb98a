"""Shared fixtures.  ``gpu`` tests need a CUDA device and the sm_100a library."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device + built sm_100a library)")


def load_cases(name, prefix):
    """Unpack a golden npz written by scripts/make_golden.py into a list of dicts."""
    with np.load(os.path.join(GOLDEN, name)) as z:
        count = int(z[f"{prefix}_count"])
        cases = [dict() for _ in range(count)]
        for key in z.files:
            if key == f"{prefix}_count":
                continue
            head, field = key.split("_", 1)
            cases[int(head[len(prefix):])][field] = z[key]
    for case in cases:
        for k, v in list(case.items()):
            if v.shape == ():
                case[k] = v.item()
    return cases


@pytest.fixture(scope="session")
def golden():
    return load_cases
