"""Generate tests/golden/fullsize_config{K}.npz: the numpy oracle's solution summary for
BASELINE configs 2 and 4 at FULL size (the GPU parity tests compare against it).

The oracle runs the factor-space Newton route (oracle.newton_direction_factor, pinned to
the reference's newton_direction goldens in tests/test_oracle_golden.py) with the
product's delta line search and the product's options (config 2: max_inner=200,
DESIGN.md section 11).  Stored: objective, R_KKT, counts, the free set J of the returned
x (reference classifier), and x summaries (sum, norm, a sample of 4096 entries).

    python scripts/make_fullsize_fixtures.py 4      # ~minutes on 8 cores
    python scripts/make_fullsize_fixtures.py 2      # ~1 h (matrix-free CG on the CPU)
"""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_1910_01312_b200 import datagen  # noqa: E402


def problem(k, cfg):
    if "indptr" in cfg:
        return O.csvc_problem_csr(cfg["indptr"], cfg["indices"], cfg["data"], cfg["shape"],
                                  cfg["y"], cfg["C"])
    if cfg["task"] == "svr":
        return O.svr_problem(cfg["A"], cfg["t"], cfg["C"], cfg["epsilon"])
    return O.csvc_problem(cfg["A"], cfg["y"], cfg["C"])


def main():
    k = int(sys.argv[1])
    t0 = time.time()
    cfg = datagen.make_config(k)
    op, c, bl = problem(k, cfg)
    O.set_psi_mode("delta")
    ssn = O.SsnOpts(newton="factor", max_inner=200 if "indptr" in cfg else 50)
    trace = []
    rep = O.alm_solve(op, c, bl, O.AlmOpts(tol_kkt=1e-6), ssn,
                      callback=lambda *a: (trace.append(a), print(a, time.time() - t0,
                                                                  flush=True)))
    x = rep["x_opt"]
    res, pr, qx = O.kkt_full(x, op, c, bl)
    J = np.flatnonzero(pr[2]).astype(np.int64)
    rng = np.random.default_rng(1234)
    sample = np.sort(rng.choice(x.size, size=min(4096, x.size), replace=False))
    out = os.path.join(ROOT, "tests", "golden", f"fullsize_config{k}.npz")
    np.savez_compressed(
        out, config=k, objective=rep["objective"], kkt=rep["kkt_residual"],
        kkt_check=res, outer=rep["outer_iters"], inner=rep["total_inner_iters"],
        p=rep["unbounded_support_count"], converged=rep["converged"], J=J,
        x_sum=float(x.sum()), x_norm=float(np.linalg.norm(x)), sample_idx=sample,
        x_sample=x[sample], trace=np.array(trace, dtype=np.float64),
        seconds=time.time() - t0)
    print(json.dumps({"config": k, "objective": rep["objective"], "kkt": rep["kkt_residual"],
                      "outer": rep["outer_iters"], "inner": rep["total_inner_iters"],
                      "p": rep["unbounded_support_count"], "J": int(J.size),
                      "seconds": time.time() - t0}))


if __name__ == "__main__":
    main()
