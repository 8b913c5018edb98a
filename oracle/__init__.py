"""CPU oracle for the SSsNAL hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the reference algorithm of arXiv 1910.01312
as implemented by the reference package (``ssnal``: projection.py, solver.py,
kernels.py, svm.py).  It is the checker for the CUDA product path and the
``cpu_baseline`` / ``--impl reference`` arm of ``bench.py``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import it.  The product package ``paper_1910_01312_b200`` never does:
it has no CPU fallback and fails loudly without its CUDA library.

Parity pinning: ``tests/golden/*.npz`` were produced by running the real
reference package (``scripts/make_golden.py``, which imports it from
/root/reference in the build container); ``tests/test_oracle_golden.py``
checks this restatement against every one of those vectors.
"""

from .ssnal_oracle import *  # noqa: F401,F403
