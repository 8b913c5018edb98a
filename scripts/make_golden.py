"""Generate tests/golden/*.npz by running the REAL reference package.

Run in the build container (where /root/reference exists):

    python scripts/make_golden.py

The reference is imported from /root/reference/pkg/src; nothing here is
needed at test time (the fixtures are committed).  Cases cover every hot-path
function the product replaces: projection (incl. zero a_i, duplicate and flat
breakpoints, all-zero a, already-feasible, SVM-shaped large n), HS-Jacobian,
the reduced Newton direction, the KKT residual, and end-to-end alm_solve on
dense QPs, linear C-SVC (incl. BASELINE config 0) and eps-SVR.
"""

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "tests", "golden")
sys.path.insert(0, REF_SRC)
sys.path.insert(0, os.path.join(HERE, ".."))

import ssnal  # noqa: E402  (the reference)
from paper_1910_01312_b200 import datagen  # noqa: E402


def rand_box_line(rng, n, zero_prob=0.15):
    a = rng.standard_normal(n)
    a[rng.random(n) < zero_prob] = 0.0
    l = -rng.random(n) - 0.1
    u = rng.random(n) + 0.1
    d = float(a.dot(l + rng.random(n) * (u - l)))
    return a, d, l, u


def pack(prefix, cases):
    """Flatten a list of dicts of arrays into one npz namespace."""
    out = {f"{prefix}_count": np.array(len(cases))}
    for i, case in enumerate(cases):
        for k, v in case.items():
            out[f"{prefix}{i}_{k}"] = np.asarray(v)
    return out


def projection_cases():
    rng = np.random.default_rng(20260101)
    cases = []
    for _ in range(80):
        n = int(rng.integers(1, 60))
        a, d, l, u = rand_box_line(rng, n)
        v = rng.standard_normal(n) * rng.choice([0.5, 2.0, 10.0])
        cases.append((v, a, d, l, u))
    # hand cases from the reference test suite's shapes
    cases.append((np.array([0.5, 0.5]), np.ones(2), 1.0, np.zeros(2), np.ones(2)))
    cases.append((np.array([2.0, 0.0]), np.ones(2), 1.0, np.zeros(2), np.ones(2)))
    cases.append((np.array([0.9, 0.8]), np.ones(2), 1.0, np.zeros(2), np.ones(2)))
    cases.append((np.array([2.0, -1.0]), np.ones(2), 1.0, np.zeros(2), np.ones(2)))
    cases.append((np.full(4, 0.6), np.ones(4), 1.0, np.zeros(4), np.ones(4)))
    cases.append((np.array([-1.0, 0.5, 9.0]), np.zeros(3), 0.0, np.zeros(3), np.ones(3)))
    # duplicated breakpoints at scale: many identical coordinates
    v = np.repeat(rng.standard_normal(7), 300)
    a = np.tile(np.array([1.0, -1.0, 1.0]), 700)
    cases.append((v, a, 0.0, np.zeros(2100), np.full(2100, 0.7)))
    # SVM-shaped: a = y (+-1), l = 0, u = C, d = 0
    for n, C, scale in ((5000, 1.0, 3.0), (20000, 0.1, 1.0), (3000, 64.0, 50.0)):
        y = np.where(rng.random(n) < 0.5, 1.0, -1.0)
        v = C * (0.5 + scale * rng.standard_normal(n))
        cases.append((v, y, 0.0, np.zeros(n), np.full(n, C)))
    # SVR-shaped: a = (e; -e)
    m = 2500
    a = np.concatenate([np.ones(m), -np.ones(m)])
    cases.append((rng.standard_normal(2 * m), a, 0.0, np.zeros(2 * m), np.ones(2 * m)))
    out = []
    for v, a, d, l, u in cases:
        s = ssnal.BoxLineSet(a=a, d=d, l=l, u=u)
        r = ssnal.project_box_line(v, s)
        m = r.active_mask
        out.append({"v": v, "a": a, "d": d, "l": l, "u": u, "x": r.x,
                    "lam": r.lambda_hat, "free": m.free_mask.astype(np.uint8),
                    "bp": ssnal.breakpoints(v, s),
                    "gphi0": ssnal.grad_phi(0.0, v, s)})
    return out


def hs_cases():
    rng = np.random.default_rng(7)
    out = []
    for _ in range(30):
        n = int(rng.integers(2, 80))
        a, d, l, u = rand_box_line(rng, n, zero_prob=0.1)
        s = ssnal.BoxLineSet(a=a, d=d, l=l, u=u)
        r = ssnal.project_box_line(rng.standard_normal(n) * 2, s)
        y = rng.standard_normal(n)
        out.append({"a": a, "free": r.active_mask.free_mask.astype(np.uint8), "y": y,
                    "py": ssnal.hs_jacobian_apply(r.active_mask, a, y)})
    return out


def random_qp(seed, n_lo=5, n_hi=40):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(n_lo, n_hi + 1))
    k = int(rng.integers(2, max(3, n // 2 + 1))) if seed % 2 == 0 else n
    g = rng.standard_normal((k, n))
    a, d, l, u = rand_box_line(rng, n)
    return g, rng.standard_normal(n), a, d, l, u


def newton_cases():
    out = []
    opts = ssnal.SsnOptions()
    seed = 100
    while len(out) < 30:
        seed += 1
        g, c, a, d, l, u = random_qp(seed, 4, 16)
        q = g.T @ g
        problem = ssnal.QpProblem(q_op=ssnal.DenseOperator(q), c=c,
                                  constraint=ssnal.BoxLineSet(a=a, d=d, l=l, u=u))
        rng = np.random.default_rng(seed)
        sigma = float(rng.choice([0.5, 1.0, 3.0, 10.0]))
        x = rng.standard_normal(q.shape[0])
        w = rng.standard_normal(q.shape[0])
        qw = q @ w
        uu = x - sigma * (qw + c)
        proj = ssnal.project_box_line(uu, problem.constraint)
        s = w - proj.x
        grad = q @ s
        if np.linalg.norm(grad) < 1e-10:
            continue
        direction, q_dir, dqd = ssnal.newton_direction(s, grad, proj, sigma, problem, opts)
        out.append({"G": g, "c": c, "a": a, "d": d, "l": l, "u": u, "sigma": sigma,
                    "x": x, "w": w, "free": proj.active_mask.free_mask.astype(np.uint8),
                    "dir": direction, "qdir": q_dir, "dqd": dqd})
    return out


def report_dict(rep):
    return {"x_opt": rep.x_opt, "kkt": rep.kkt_residual, "outer": rep.outer_iters,
            "inner": rep.total_inner_iters, "p": rep.unbounded_support_count,
            "obj": rep.objective, "converged": rep.converged}


def solve_cases():
    out = []
    # tiny instance (n=2, Q=I, c=-e, a=e, d=1, box [0,1]^2)
    tiny = ssnal.QpProblem(q_op=ssnal.DenseOperator(np.eye(2)), c=-np.ones(2),
                           constraint=ssnal.BoxLineSet(a=np.ones(2), d=1.0,
                                                       l=np.zeros(2), u=np.ones(2)))
    rep = ssnal.alm_solve(tiny, ssnal.AlmOptions(tol_kkt=1e-10))
    out.append({"kind": "dense", "G": np.eye(2), "c": -np.ones(2), "a": np.ones(2),
                "d": 1.0, "l": np.zeros(2), "u": np.ones(2), "tol": 1e-10,
                **report_dict(rep)})
    for seed in range(200, 210):
        g, c, a, d, l, u = random_qp(seed)
        problem = ssnal.QpProblem(q_op=ssnal.DenseOperator(g.T @ g), c=c,
                                  constraint=ssnal.BoxLineSet(a=a, d=d, l=l, u=u))
        rep = ssnal.alm_solve(problem, ssnal.AlmOptions(tol_kkt=1e-8))
        out.append({"kind": "dense", "G": g, "c": c, "a": a, "d": d, "l": l, "u": u,
                    "tol": 1e-8, **report_dict(rep)})
    # linear C-SVC: small planted set, and BASELINE config 0 (n=2000, q=50)
    rng = np.random.default_rng(5)
    a_s = rng.standard_normal((300, 8))
    y_s = np.sign(a_s @ rng.standard_normal(8) + 0.3 * rng.standard_normal(300))
    y_s[y_s == 0] = 1.0
    cfg0 = datagen.config0()
    for a_mat, y, C, tol in ((a_s, y_s, 1.0, 1e-8), (cfg0["A"], cfg0["y"], 1.0, 1e-6)):
        config = ssnal.SvmConfig(task="classification", C=C)
        problem = ssnal.build_csvc_dual(a_mat, y, config)
        rep = ssnal.alm_solve(problem, ssnal.AlmOptions(tol_kkt=tol))
        out.append({"kind": "csvc", "A": a_mat, "y": y, "C": C, "tol": tol,
                    **report_dict(rep)})
    # eps-SVR, linear kernel
    rng = np.random.default_rng(9)
    a_r = rng.standard_normal((150, 5))
    t_r = a_r @ (rng.standard_normal(5) / np.sqrt(5)) + 0.1 * rng.standard_normal(150)
    config = ssnal.SvmConfig(task="regression", C=1.0, epsilon=0.1)
    problem = ssnal.build_svr_dual(a_r, t_r, config)
    rep = ssnal.alm_solve(problem, ssnal.AlmOptions(tol_kkt=1e-8))
    out.append({"kind": "svr", "A": a_r, "t": t_r, "C": 1.0, "eps": 0.1, "tol": 1e-8,
                **report_dict(rep)})
    return out


def kkt_cases():
    out = []
    for seed in range(300, 306):
        g, c, a, d, l, u = random_qp(seed)
        problem = ssnal.QpProblem(q_op=ssnal.DenseOperator(g.T @ g), c=c,
                                  constraint=ssnal.BoxLineSet(a=a, d=d, l=l, u=u))
        x = np.random.default_rng(seed).standard_normal(g.shape[1])
        out.append({"G": g, "c": c, "a": a, "d": d, "l": l, "u": u, "x": x,
                    "kkt": ssnal.kkt_residual(x, problem)})
    return out


def svm_cases():
    """The reference's train / recover_bias / decision_function / evaluate (svm.py:147-295)
    on linear C-SVC and eps-SVR sets, plus bound-only duals (interval-midpoint branch)."""
    out = []
    rng = np.random.default_rng(77)
    cfg0 = datagen.config0()
    a_s = rng.standard_normal((300, 8))
    y_s = np.sign(a_s @ rng.standard_normal(8) + 0.3 * rng.standard_normal(300))
    y_s[y_s == 0] = 1.0
    a_r = rng.standard_normal((200, 6))
    t_r = a_r @ (rng.standard_normal(6) / np.sqrt(6)) + 0.1 * rng.standard_normal(200)
    sets = [("classification", a_s, y_s, 1.0, 0.0, 1e-8),
            ("classification", cfg0["A"], cfg0["y"], 1.0, 0.0, 1e-6),
            ("regression", a_r, t_r, 1.0, 0.1, 1e-8),
            ("regression", a_r, t_r, 0.5, 0.3, 1e-8)]
    for task, feats, targ, C, eps, tol in sets:
        config = ssnal.SvmConfig(task=task, C=C, epsilon=eps)
        model, rep = ssnal.train(feats, targ, config, alm_opts=ssnal.AlmOptions(tol_kkt=tol))
        pts = feats[::7]
        metric = ssnal.evaluate(model, feats, targ)
        out.append({"task": task, "A": feats, "t": targ, "C": C, "eps": eps, "tol": tol,
                    "dual_x": model.dual_x, "bias": model.bias,
                    "support_indices": model.support_indices,
                    "support_coef": model.support_coef,
                    "decision": ssnal.decision_function(model, pts), "points": pts,
                    "metric": list(metric.values())[0]})
    # no free dual: the bias is the midpoint of the bound-active interval
    n = 40
    a_b = rng.standard_normal((n, 3))
    y_b = np.where(rng.random(n) < 0.5, 1.0, -1.0)
    x_b = np.where(rng.random(n) < 0.5, 0.0, 1.0)
    cfg = ssnal.SvmConfig(task="classification", C=1.0)
    out.append({"task": "classification", "A": a_b, "t": y_b, "C": 1.0, "eps": 0.0,
                "tol": 0.0, "dual_x": x_b, "bias": ssnal.recover_bias(x_b, a_b, y_b, cfg),
                "support_indices": np.flatnonzero(x_b), "support_coef": x_b[x_b > 0],
                "decision": np.zeros(1), "points": a_b[:1], "metric": 0.0})
    t_b = a_b @ np.ones(3)
    xz = np.where(rng.random(2 * n) < 0.5, 0.0, 0.5)
    cfg = ssnal.SvmConfig(task="regression", C=0.5, epsilon=0.2)
    out.append({"task": "regression", "A": a_b, "t": t_b, "C": 0.5, "eps": 0.2, "tol": 0.0,
                "dual_x": xz, "bias": ssnal.recover_bias(xz, a_b, t_b, cfg),
                "support_indices": np.zeros(0, np.int64), "support_coef": np.zeros(0),
                "decision": np.zeros(1), "points": a_b[:1], "metric": 0.0})
    return out


def main():
    os.makedirs(OUT, exist_ok=True)
    if "--svm-only" in sys.argv:
        np.savez_compressed(os.path.join(OUT, "svm.npz"), **pack("v", svm_cases()))
        print("wrote svm.npz")
        return
    np.savez_compressed(os.path.join(OUT, "projection.npz"), **pack("p", projection_cases()))
    np.savez_compressed(os.path.join(OUT, "hs_jacobian.npz"), **pack("h", hs_cases()))
    np.savez_compressed(os.path.join(OUT, "newton.npz"), **pack("n", newton_cases()))
    np.savez_compressed(os.path.join(OUT, "kkt.npz"), **pack("k", kkt_cases()))
    np.savez_compressed(os.path.join(OUT, "solve.npz"), **pack("s", solve_cases()))
    np.savez_compressed(os.path.join(OUT, "svm.npz"), **pack("v", svm_cases()))
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
