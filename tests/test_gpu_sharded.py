"""Row-sharded path on the GPU: the shard-local kernels of csrc/dist.cu against the
single-GPU projection; the NATIVE sharded driver (ssnal_alm_solve_sharded) with 2 and 3
ranks as threads on this one GPU (loopback transport: host-ordered collectives, no
kernel waits on another rank) and with 1 rank over NCCL, against the single-GPU
driver, the golden reference runs and an independent KKT certificate; the Python
mirror of the sharded engine over NCCL.  (The gloo multi-rank runs of the Python
mirror are tests/test_sharded_cpu.py.)"""

import os
import socket

import numpy as np
import pytest
import torch

from conftest import load_cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import __graft_entry__ as g

    g.build()
    import paper_1910_01312_b200 as P

    return P


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_proj_local_slices_fold_to_the_full_projection(pkg):
    """Two slices evaluated separately and folded in order == the whole vector."""
    from paper_1910_01312_b200 import _lib, projection
    from paper_1910_01312_b200.backend import default_backend

    be = default_backend()
    rng = np.random.default_rng(5)
    n = 100_003
    a = np.where(rng.random(n) < 0.5, 1.0, -1.0)
    v = rng.standard_normal(n) * 2.0
    box = projection.BoxLineSet(a, 0.0, np.zeros(n), np.ones(n))
    st = be.new_states(1)
    x_full = be.empty(n)
    f_full = be.zeros(n, torch.uint8)
    vd = torch.from_numpy(v).cuda()
    be.project(vd, box, st, 1, x_out=x_full, free_out=f_full)
    rec_full = be.read_states(st.cpu())[0]
    lam = float(rec_full["lam"])
    cut = 37_001
    parts = []
    xs = []
    for lo, hi in ((0, cut), (cut, n)):
        sub = projection.BoxLineSet(a[lo:hi], 0.0, np.zeros(hi - lo), np.ones(hi - lo))
        rec = be.zeros(16)
        be.proj_local(vd[lo:hi], sub, 1, [lam], 0, rec)
        ev = rec[:5].cpu().numpy().copy()
        xo = be.empty(hi - lo)
        be.proj_local(vd[lo:hi], sub, 1, [lam], 1, rec, x_out=xo)
        parts.append((ev, rec[:6].cpu().numpy().copy()))
        xs.append(xo.cpu().numpy())
    f = parts[0][0][0] + parts[1][0][0]
    assert abs(f) <= 1e-10 * np.abs(a).sum()  # a'x(lambda*) = d = 0
    assert min(parts[0][0][3], parts[1][0][3]) > lam > max(parts[0][0][4], parts[1][0][4])
    np.testing.assert_array_equal(np.concatenate(xs), x_full.cpu().numpy())
    sums = parts[0][1] + parts[1][1]
    assert sums[3] == pytest.approx(rec_full["sum_a2_free"], rel=1e-12)
    assert int(round(sums[4])) == int(rec_full["nfree"])
    assert sums[5] == pytest.approx(rec_full["sum_xv"], rel=1e-12)


def test_sum_slices_and_hs_apply_coef(pkg):
    from paper_1910_01312_b200.backend import default_backend

    be = default_backend()
    rng = np.random.default_rng(2)
    src = torch.from_numpy(rng.standard_normal((3, 1001))).cuda()
    out = be.empty(1001)
    be.sum_slices(3, src, out)
    h = src.cpu().numpy()
    np.testing.assert_array_equal(out.cpu().numpy(), (h[0] + h[1]) + h[2])
    n = 5000
    free = torch.from_numpy((rng.random(n) < 0.4).astype(np.uint8)).cuda()
    a, y, s = (torch.from_numpy(rng.standard_normal(n)).cuda() for _ in range(3))
    o = be.empty(n)
    be.hs_apply_coef(free, a, y, -2.0, s, -1.0, 0.3, o)
    fm = free.cpu().numpy().astype(bool)
    ref = -s.cpu().numpy() - 2.0 * np.where(fm, y.cpu().numpy() - 0.3 * a.cpu().numpy(), 0.0)
    np.testing.assert_allclose(o.cpu().numpy(), ref, rtol=1e-15, atol=1e-15)


def test_sharded_world1_nccl_matches_native(pkg):
    import torch.distributed as dist

    from paper_1910_01312_b200 import datagen, sharded

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        comm = sharded.ShardComm()
        for c in load_cases("solve.npz", "s"):
            if c["kind"] == "dense":
                continue
            if c["kind"] == "csvc":
                pb = sharded.build_csvc_dual_sharded(c["A"], c["y"], c["C"], comm)
            else:
                pb = sharded.build_svr_dual_sharded(c["A"], c["t"], c["C"], c["eps"], comm)
            rep = pkg.alm_solve(pb, pkg.AlmOptions(tol_kkt=c["tol"]))
            assert rep.converged and rep.kkt_residual < c["tol"]
            assert (rep.outer_iters, rep.total_inner_iters) == (c["outer"], c["inner"])
            assert rep.objective == pytest.approx(c["obj"], rel=1e-6, abs=1e-9)
            x = sharded.gather_solution(pb, rep.x_opt)
            np.testing.assert_allclose(x, c["x_opt"], atol=1e-6)
        cfg = datagen.config1(seed=3, n=8000, q=120)
        pb = sharded.build_csvc_dual_sharded(cfg["A"], cfg["y"], cfg["C"], comm)
        rep = pkg.alm_solve(pb, pkg.AlmOptions(tol_kkt=1e-6))
        nat = pkg.alm_solve(pkg.build_csvc_dual(cfg["A"], cfg["y"], cfg["C"]),
                            pkg.AlmOptions(tol_kkt=1e-6))
        assert rep.converged and nat.converged
        assert rep.objective == pytest.approx(nat.objective, rel=1e-6)
        # sparse operator (config-3 generator, Zipf columns): rank-local CSR products and
        # the sharded factor-space CG vs the single-GPU native driver
        cfg = datagen.make_config(3, n=6000, q=3000)
        csr = (cfg["indptr"], cfg["indices"], cfg["data"], cfg["shape"])
        pb = sharded.build_csvc_dual_sharded(csr, cfg["y"], cfg["C"], comm)
        ssn = pkg.SsnOptions(max_inner=200)
        rep = pkg.alm_solve(pb, pkg.AlmOptions(tol_kkt=1e-6), ssn)
        nat = pkg.alm_solve(pkg.build_csvc_dual(csr, cfg["y"], cfg["C"]),
                            pkg.AlmOptions(tol_kkt=1e-6), ssn)
        assert rep.converged and nat.converged and rep.kkt_residual <= 1e-6
        assert pb.native_counters["cg_iters"] > 0  # the native sharded factor-space CG
        assert rep.objective == pytest.approx(nat.objective, rel=1e-6)
        # the Python mirror of the sharded engine on the same group
        cfg = datagen.config1(seed=4, n=4000, q=60)
        pb = sharded.build_csvc_dual_sharded(cfg["A"], cfg["y"], cfg["C"], comm)
        rep = pkg.alm_solve(pb, pkg.AlmOptions(tol_kkt=1e-6), pkg.SsnOptions(engine="python"))
        nat = pkg.alm_solve(pkg.build_csvc_dual(cfg["A"], cfg["y"], cfg["C"]),
                            pkg.AlmOptions(tol_kkt=1e-6))
        assert rep.converged and rep.objective == pytest.approx(nat.objective, rel=1e-6)
        comm.close()
    finally:
        dist.destroy_process_group()


# ------------------------------------------------------------ native sharded, loopback
def _assemble(kind, reps, sizes):
    """Global dual vector (reference ordering) from the ranks' slices."""
    parts = [np.asarray(r.x_opt) for r in reps]
    if kind == "csvc":
        return np.concatenate(parts)
    return np.concatenate([np.concatenate([p[:m] for p, m in zip(parts, sizes)]),
                           np.concatenate([p[m:] for p, m in zip(parts, sizes)])])


def _check_ranks_agree(reps):
    """Every rank holds the same reduced scalars: identical reports."""
    for r in reps[1:]:
        assert (r.kkt_residual, r.objective, r.outer_iters, r.total_inner_iters,
                r.unbounded_support_count) == (reps[0].kkt_residual, reps[0].objective,
                                               reps[0].outer_iters, reps[0].total_inner_iters,
                                               reps[0].unbounded_support_count)


@pytest.mark.parametrize("world", [2, 3])
def test_native_sharded_loopback_csvc(pkg, world):
    from paper_1910_01312_b200 import datagen, sharded

    cfg = datagen.config1(seed=11, n=12000, q=80)
    A, y, C = cfg["A"], cfg["y"], cfg["C"]
    single = pkg.build_csvc_dual(A, y, C)
    nat = pkg.alm_solve(single, pkg.AlmOptions(tol_kkt=1e-6))
    cuts = [sharded.shard_range(A.shape[0], r, world) for r in range(world)]
    probs = [pkg.build_csvc_dual(A[lo:hi], y[lo:hi], C) for lo, hi in cuts]
    reps = sharded.solve_loopback(probs, pkg.AlmOptions(tol_kkt=1e-6))
    _check_ranks_agree(reps)
    rep = reps[0]
    assert rep.converged and rep.kkt_residual <= 1e-6
    assert rep.objective == pytest.approx(nat.objective, rel=1e-8)
    x = _assemble("csvc", reps, [hi - lo for lo, hi in cuts])
    assert pkg.kkt_residual(x, single) <= 1e-6  # certified by the single-GPU operator
    assert abs(float(np.dot(y, x))) <= 1e-9 * (1 + np.abs(x).sum())
    assert x.min() >= 0.0 and x.max() <= C
    np.testing.assert_allclose(x, nat.x_opt, atol=1e-5)
    assert rep.unbounded_support_count == nat.unbounded_support_count


@pytest.mark.parametrize("world", [2, 3])
def test_native_sharded_loopback_svr(pkg, world):
    from paper_1910_01312_b200 import datagen, sharded

    cfg = datagen.make_config(4, n=20000, q=50)
    A, t = cfg["A"], cfg["t"]
    single = pkg.build_svr_dual(A, t, cfg["C"], cfg["epsilon"])
    nat = pkg.alm_solve(single, pkg.AlmOptions(tol_kkt=1e-6))
    cuts = [sharded.shard_range(A.shape[0], r, world) for r in range(world)]
    probs = [pkg.build_svr_dual(A[lo:hi], t[lo:hi], cfg["C"], cfg["epsilon"]) for lo, hi in cuts]
    reps = sharded.solve_loopback(probs, pkg.AlmOptions(tol_kkt=1e-6))
    _check_ranks_agree(reps)
    rep = reps[0]
    assert rep.converged and rep.kkt_residual <= 1e-6
    assert rep.objective == pytest.approx(nat.objective, rel=1e-8)
    x = _assemble("svr", reps, [hi - lo for lo, hi in cuts])
    assert pkg.kkt_residual(x, single) <= 1e-6
    np.testing.assert_allclose(x, nat.x_opt, atol=1e-5)


@pytest.mark.parametrize("q", [1500, 3000])
def test_native_sharded_loopback_csr(pkg, q):
    """Config-3 generator (Zipf columns): q <= 2048 runs the all-reduced q x q direct
    system, q > 2048 the sharded factor-space Jacobi CG."""
    from paper_1910_01312_b200 import datagen, sharded

    cfg = datagen.make_config(3, n=8000, q=q)
    indptr, indices, data = cfg["indptr"], cfg["indices"], cfg["data"]
    y, C = cfg["y"], cfg["C"]
    single = pkg.build_csvc_dual((indptr, indices, data, cfg["shape"]), y, C)
    ssn = pkg.SsnOptions(max_inner=200)
    nat = pkg.alm_solve(single, pkg.AlmOptions(tol_kkt=1e-6), ssn)
    world = 2
    cuts = [sharded.shard_range(len(y), r, world) for r in range(world)]
    probs = []
    for lo, hi in cuts:
        ip = np.asarray(indptr[lo:hi + 1]) - indptr[lo]
        sl = slice(int(indptr[lo]), int(indptr[hi]))
        probs.append(pkg.build_csvc_dual((ip, indices[sl], data[sl], (hi - lo, q)), y[lo:hi], C))
    reps = sharded.solve_loopback(probs, pkg.AlmOptions(tol_kkt=1e-6), ssn)
    _check_ranks_agree(reps)
    rep = reps[0]
    assert rep.converged and rep.kkt_residual <= 1e-6
    assert rep.objective == pytest.approx(nat.objective, rel=1e-6)
    x = _assemble("csvc", reps, [hi - lo for lo, hi in cuts])
    assert pkg.kkt_residual(x, single) <= 1e-6
    if q > 2048:
        assert probs[0].native_counters["cg_iters"] > 0
