"""Row-sharded path on the GPU: the shard-local kernels of csrc/dist.cu against the
single-GPU projection, and the sharded solver at world size 1 over NCCL against the
native driver and the golden reference runs.  (world > 1 needs more than the one
GPU a gpurun box has; the multi-rank control flow is covered over gloo in
tests/test_sharded_cpu.py.)"""

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
        cfg = datagen.make_config(3, n=6000, q=1500)
        csr = (cfg["indptr"], cfg["indices"], cfg["data"], cfg["shape"])
        pb = sharded.build_csvc_dual_sharded(csr, cfg["y"], cfg["C"], comm)
        ssn = pkg.SsnOptions(max_inner=200)
        rep = pkg.alm_solve(pb, pkg.AlmOptions(tol_kkt=1e-6), ssn)
        nat = pkg.alm_solve(pkg.build_csvc_dual(csr, cfg["y"], cfg["C"]),
                            pkg.AlmOptions(tol_kkt=1e-6), ssn)
        assert rep.converged and nat.converged and rep.kkt_residual <= 1e-6
        assert pb.engine().counters.get("cg_iters", 0) > 0
        assert rep.objective == pytest.approx(nat.objective, rel=1e-6)
    finally:
        dist.destroy_process_group()
