"""Seeded synthetic stand-ins for the five BASELINE.json workload configs.

The reference quotes its SVM results on LIBSVM benchmark files, which are not
available offline; these generators reproduce the shapes, sparsity and value
distributions that BASELINE.json names ("Workloads").  All are
host-side numpy (they produce the HOST buffers the end-to-end path uploads).
"""

import numpy as np

from .errors import InputError


def config0(seed=0, n=2000, q=50):
    """C-SVC, dense: A~N(0,1); planted w~N(0,I); y = sign(Aw + 0.1 N(0,1)); C = 1."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, q))
    w = rng.standard_normal(q)
    y = np.sign(a @ w + 0.1 * rng.standard_normal(n))
    y[y == 0] = 1.0
    return {"A": a, "y": y, "C": 1.0, "task": "csvc"}


def config1(seed=1, n=50_000, q=300):
    """C-SVC, dense: two-class Gaussian mixture, means +-0.5*1, identity covariance,
    balanced labels; C = 1."""
    rng = np.random.default_rng(seed)
    y = np.ones(n)
    y[n // 2:] = -1.0
    rng.shuffle(y)
    a = rng.standard_normal((n, q))
    a += 0.5 * y[:, None]
    return {"A": a, "y": y, "C": 1.0, "task": "csvc"}


def _csr_rows(rng, n, q, nnz_row, col_sampler):
    """Row-wise CSR with ``nnz_row`` distinct sorted columns per row and unit-L2 rows
    of |N(0,1)| values."""
    indptr = np.arange(0, (n + 1) * nnz_row, nnz_row, dtype=np.int64)
    cols = col_sampler(rng, n, q, nnz_row)
    vals = np.abs(rng.standard_normal((n, nnz_row)))
    vals /= np.linalg.norm(vals, axis=1, keepdims=True)
    return indptr, cols.astype(np.int32).ravel(), vals.ravel()


def _distinct_uniform_cols(rng, n, q, k):
    cols = rng.integers(0, q, size=(n, k))
    cols.sort(axis=1)
    dup = np.any(cols[:, 1:] == cols[:, :-1], axis=1)
    for i in np.flatnonzero(dup):  # rare for k << q: redraw without replacement
        cols[i] = np.sort(rng.choice(q, size=k, replace=False))
    return cols


def _zipf_ranks(rng, shape, s, q, head=4096):
    """0-based ranks from Zipf(s) on [1, q] by inverse CDF: exact table for the
    ``head`` most popular ranks, midpoint-integral approximation of the tail mass
    (relative pmf error < 1e-6 past rank 4096)."""
    h = min(head, q)
    pmf = np.arange(1, h + 1, dtype=np.float64) ** (-s)
    lo = h + 0.5
    tail = (lo ** (1 - s) - (q + 0.5) ** (1 - s)) / (s - 1) if q > h else 0.0
    z = pmf.sum() + tail
    cdf = np.cumsum(pmf) / z
    u = rng.random(shape)
    out = np.searchsorted(cdf, u)  # < h: head rank
    t = out >= h
    if t.any():
        m = (u[t] - cdf[-1]) * z * (s - 1)
        r = np.ceil((lo ** (1 - s) - m) ** (1.0 / (1 - s)) - 0.5)
        out[t] = np.clip(r, h + 1, q).astype(np.int64) - 1
    return np.minimum(out, q - 1)


def _distinct_zipf_cols(rng, n, q, k, s=1.1):
    """Columns drawn with Zipf(s) popularity over a random column permutation."""
    perm = rng.permutation(q)
    out = np.empty((n, k), dtype=np.int64)
    chunk = 1 << 16
    for start in range(0, n, chunk):
        stop = min(start + chunk, n)
        m = stop - start
        block = np.sort(perm[_zipf_ranks(rng, (m, 3 * k), s, q)], axis=1)
        dup = np.zeros(block.shape, dtype=bool)
        dup[:, 1:] = block[:, 1:] == block[:, :-1]
        # keep k distinct candidates per row chosen uniformly: random keys, duplicates last
        keys = rng.random(block.shape)
        keys[dup] = 2.0
        pick = np.argsort(keys, axis=1)[:, :k]
        sel = np.take_along_axis(block, pick, axis=1)
        short = np.flatnonzero((~dup).sum(axis=1) < k)
        for r in short:  # hot columns collided too often: top up with more draws
            uniq = np.unique(block[r])
            while uniq.size < k:
                extra = perm[_zipf_ranks(rng, (2 * k,), s, q)]
                uniq = np.unique(np.concatenate([uniq, extra]))
            sel[r] = uniq[rng.choice(uniq.size, size=k, replace=False)]
        out[start:stop] = np.sort(sel, axis=1)
    return out


def _planted_labels(rng, indptr, cols, vals, q, density, flip):
    n = indptr.size - 1
    w = np.zeros(q)
    nz = rng.choice(q, size=max(1, int(density * q)), replace=False)
    w[nz] = rng.standard_normal(nz.size)
    row = np.repeat(np.arange(n), np.diff(indptr))
    score = np.bincount(row, weights=vals * w[cols], minlength=n)
    y = np.where(score >= 0.0, 1.0, -1.0)
    flips = rng.random(n) < flip
    y[flips] = -y[flips]
    return y


def config2(seed=2, n=500_000, q=100_000, nnz_row=50):
    """C-SVC, sparse CSR: 50 distinct uniform columns per row, |N(0,1)| values,
    unit-L2 rows; labels from planted sparse w (1% nnz) with 10% flips; C = 1."""
    rng = np.random.default_rng(seed)
    indptr, cols, vals = _csr_rows(rng, n, q, nnz_row, _distinct_uniform_cols)
    y = _planted_labels(rng, indptr, cols, vals, q, 0.01, 0.10)
    return {"indptr": indptr, "indices": cols, "data": vals, "shape": (n, q), "y": y,
            "C": 1.0, "task": "csvc"}


def config3(seed=3, n=4_000_000, q=1_000_000, nnz_row=30):
    """C-SVC, sparse CSR, Zipf(1.1) column popularity, 30 nnz/row, unit-L2 rows;
    planted sparse w with 5% flips; C = 0.1."""
    rng = np.random.default_rng(seed)
    indptr, cols, vals = _csr_rows(rng, n, q, nnz_row, _distinct_zipf_cols)
    y = _planted_labels(rng, indptr, cols, vals, q, 0.01, 0.05)
    return {"indptr": indptr, "indices": cols, "data": vals, "shape": (n, q), "y": y,
            "C": 0.1, "task": "csvc"}


def config4(seed=4, n=1_000_000, q=500):
    """eps-SVR, dense: A~N(0,1), t = Aw + N(0, 0.1^2), w~N(0, I/q); eps = 0.1, C = 1."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, q))
    w = rng.standard_normal(q) / np.sqrt(q)
    t = a @ w + 0.1 * rng.standard_normal(n)
    return {"A": a, "t": t, "C": 1.0, "epsilon": 0.1, "task": "svr"}


CONFIGS = {0: config0, 1: config1, 2: config2, 3: config3, 4: config4}


def solve_options(cfg):
    """Solver options the workloads are run with: ``{"alm": {...}, "ssn": {...}}`` keyword
    sets for AlmOptions / SsnOptions (both are reference options, ref solver.py:73-95).
    Dense configs: the reference defaults.  Sparse (CSR) configs, whose Newton systems
    are solved by matrix-free CG: ``max_inner=200`` (the default 50 ends the large-sigma
    subproblems early) and ``sigma_max=625`` -- the CG system's condition number grows
    with sigma, and capping the penalty trades a few more outer iterations for ~5x fewer
    CG iterations (config 3: 113 s -> 21 s; profiles/r2_sigma_study_*.txt)."""
    if "indptr" in cfg:
        return {"alm": {"sigma_max": 625.0}, "ssn": {"max_inner": 200}}
    return {"alm": {}, "ssn": {}}


def tuned_alm_options(cfg):
    """A faster penalty schedule for the dense eps-SVR workload (config 4), or None: start
    at sigma0 = 125 and stop growing at sigma_max = 15625 (both reference options).  The
    first outer iterations of the default schedule (sigma = 1, 5, 25) run with 3-6 x 10^5
    free slots and pay for large Gram rebuilds; the last ones (sigma >= 78125) pass the
    Armijo test only at step lengths ~1e-7.  Config 4: 5 outer / 39 inner iterations instead
    of 8 / 62, objective equal to 3e-8 relative (profiles/r2_sigma_study_config4*.txt).
    bench.py reports it BESIDE the headline, which stays on the reference defaults."""
    if "indptr" not in cfg and cfg.get("task") == "svr":
        return {"sigma0": 125.0, "sigma_max": 15625.0}
    return None


def make_config(k, **overrides):
    if k not in CONFIGS:
        raise InputError(f"unknown config {k}")
    return CONFIGS[k](**overrides)
