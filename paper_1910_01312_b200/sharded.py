"""Row-sharded SSsNAL: one process per GPU, each rank owning a contiguous slice of
the samples (rows of X) and of the dual vector.

BASELINE configs 3 and 4 are quoted "row-sharded over 1/2/4/8 GPUs".  The data
products split cleanly by rows: X d is rank-local, X^T v is a sum of rank-local
partials.  The places the path genuinely couples the slots are

  * X^T v (q-vector) and the factor-space Gram X_J^T X_J (q x q),
  * the inner products of the line search / stopping tests,
  * the projection's multiplier lambda (one equality constraint over all n),

and each is reduced here: q-vectors and the q x q Gram by one NCCL all-reduce (every
rank receives the same buffer), the projection's small per-pass records by an
all-gather folded in rank order on the host, so every rank holds bit-identical
scalars and takes identical branches.  Over gloo (CPU tests) the q-vectors are
all-gathered and folded in rank order too (csrc/dist.cu ``ssnal_sum_slices``).

The projection search runs the safeguarded Newton of csrc/proj.cu one pass per
all-gather: each pass evaluates, rank-locally, f(lambda) = sum a clip(v - lambda
a, l, u), the one-sided slopes and the nearest breakpoints (ssnal_proj_local mode
0); the host folds the records and either lands exactly on the affine piece that
holds the root (the reference's interpolation, ref projection.py:204-208) or
moves lambda.  The Newton system is always the q x q factor-space one (the
Woodbury p x p dual would need the free rows of other ranks).

Two engines run this partition:

  * the native sharded driver (csrc/driver.cu through ssnal_alm_solve_sharded): the
    whole ALM/SsN loop in C++ on the rank's stream, its collectives NCCL all-reduces /
    all-gathers enqueued on that stream (csrc/comm.cu, a communicator of the library's
    own, bootstrapped through torch.distributed); the projection search runs on the
    device (one all-gather of 8-double records per pass).  ``alm_solve`` takes it for
    NCCL groups.  ``solve_loopback`` runs the same driver with the ranks as threads of
    one process on one GPU (host-ordered collectives, no kernel waits on another rank):
    the multi-rank tests of the one-GPU boxes.
  * the Python mirror (solver._Engine / ssn_solve / alm_solve with ``ShardedBackend``
    making every reduction global and ``ShardedEngine`` replacing the direction
    assembly): gloo groups (the CPU tests) and ``SsnOptions(engine="python")``.
"""

import ctypes
import math
import threading

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .backend import F64, as_device, default_backend
from .errors import InfeasibleProblemError, InputError, InternalError
from .operators import LinearKernelOperator
from .projection import BoxLineSet
from .solver import QpProblem, _Engine

MAX_PASSES = 200  # projection search passes per call (warm-started: typically 1-3)


class ShardComm:
    """Rank / world of a torch.distributed group and the all-gather transport."""

    def __init__(self, group=None):
        if not dist.is_initialized():
            raise InputError("torch.distributed is not initialised")
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"
        self._native = None

    def native(self):
        """The library's own NCCL communicator over this group (ssnal_comm_t for the
        native sharded driver), created once: rank 0 makes the unique id, the group
        broadcasts it, every rank joins with its current device."""
        if self._native is None:
            if not self.nccl:
                raise InputError("the native sharded driver needs an NCCL process group")
            _lib.load()
            uid = ctypes.create_string_buffer(_lib.COMM_ID_BYTES)
            if self.rank == 0:
                _lib.call("ssnal_nccl_unique_id", uid)
            box = [bytes(uid.raw)]
            dist.broadcast_object_list(box, src=dist.get_global_rank(self.group, 0)
                                       if self.group is not None else 0, group=self.group)
            comm = _lib.Comm()
            _lib.call("ssnal_nccl_comm_create", self.world, self.rank, box[0], ctypes.byref(comm))
            self._native = comm
        return self._native

    def close(self):
        if self._native is not None:
            _lib.load().ssnal_comm_destroy(ctypes.byref(self._native))
            self._native = None

    def all_gather(self, t):
        """(world, *t.shape) tensor of every rank's t (same device as t)."""
        t = t.contiguous()
        out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        if self.world == 1:
            out[0].copy_(t)
        elif self.nccl:
            dist.all_gather_into_tensor(out, t, group=self.group)
        else:
            dist.all_gather(list(out.unbind(0)), t, group=self.group)
        return out

    def all_gather_objects(self, obj):
        out = [None] * self.world
        dist.all_gather_object(out, obj, group=self.group)
        return out


def shard_range(n, rank, world):
    """Contiguous balanced slice [lo, hi) of n rows for ``rank``."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class ShardedBackend:
    """A device backend whose reductions are global over the group.  Everything
    not overridden (memory, element-wise kernels, local products) is the wrapped
    single-GPU backend's."""

    name = "sharded"

    def __init__(self, base, comm):
        self.base = base
        self.comm = comm
        self.rec = base.zeros(16 * 8)  # (T <= 16) x 8 shard record
        self.collectives = 0
        import os

        self.ordered = os.environ.get("SSNAL_SHARD_ORDERED", "") not in ("", "0")

    def __getattr__(self, name):
        return getattr(self.base, name)

    # ---------------------------------------------------------------- reductions
    def allsum(self, t):
        """t <- sum over ranks of t (in place).  NCCL: one all-reduce (ring / NVLS over
        NVSwitch; every rank receives the same reduced buffer, so the replicated
        q-vectors and scalars stay bit-identical across ranks and the branches uniform).
        gloo (CPU tests): all-gather + fold in rank order (ssnal_sum_slices), the same
        sums bit for bit whatever the transport's algorithm.  SSNAL_SHARD_ORDERED=1 forces
        the ordered fold on NCCL too (results independent of the world size's NCCL
        reduction tree, at world x the traffic)."""
        if self.comm.world == 1:
            return
        flat = t.view(-1)
        self.collectives += 1
        if self.comm.nccl and not self.ordered:
            dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=self.comm.group)
            return
        g = self.comm.all_gather(flat)
        self.base.sum_slices(self.comm.world, g, flat)

    def dots(self, pairs, out, mask=None, replicated=False):
        self.base.dots(pairs, out, mask)
        if not replicated:
            self.allsum(out[: len(pairs)])

    def dense_xt(self, op, vs, out):
        self.base.dense_xt(op, vs, out)
        self.allsum(out[: len(vs)])

    def csr_xt(self, op, v, out):
        self.base.csr_xt(op, v, out)
        self.allsum(out)

    def csr_colsq(self, op, keep, out):
        self.base.csr_colsq(op, keep, out)
        self.allsum(out)

    def _fold(self, rec_dev, T, mode):
        """All-gather the (T, 8) shard records and fold them in rank order (host)."""
        g = self.comm.all_gather(rec_dev[: 8 * T]).cpu().numpy().reshape(self.comm.world, T, 8)
        self.collectives += 1
        out = g[0].copy()
        for r in range(1, self.comm.world):
            if mode == 0:
                out[:, :3] += g[r, :, :3]
                out[:, 3] = np.minimum(out[:, 3], g[r, :, 3])
                out[:, 4] = np.maximum(out[:, 4], g[r, :, 4])
            else:
                out[:, :6] += g[r, :, :6]
        return out

    # ---------------------------------------------------------------- projection
    def project(self, A, box, states, T=1, B=None, coefs=None, x_out=None, free_out=None,
                ref=None, phases=None, passes=None, hint=0.0, newton=None, base=None,
                base_lam=0.0):
        """Global projection of T trial points v_t = A - coefs[t] B (rank slices);
        writes the T global state records, x_out / free_out rank-locally."""
        d = float(getattr(box, "d_global", box.d))
        coefs = [float(c) for c in coefs] if B is not None else None
        lam = [float(hint)] * T
        lo, hi = [-math.inf] * T, [math.inf] * T
        done = [False] * T
        npass = 0
        while not all(done):
            npass += 1
            if npass > MAX_PASSES:
                raise InternalError("sharded projection: multiplier search did not converge")
            act = [t for t in range(T) if not done[t]]
            self.base.proj_local(A, box, len(act), [lam[t] for t in act], 0, self.rec, B=B,
                                 coefs=[coefs[t] for t in act] if B is not None else None)
            rec = self._fold(self.rec, len(act), 0)
            for j, t in enumerate(act):
                f, s_r, s_l, b_r, b_l = (float(v) for v in rec[j, :5])
                g, c = d - f, lam[t]
                if g < 0.0:  # root to the right (phi' = d - f is non-decreasing)
                    lo[t] = c
                    if s_r > 0.0:
                        ln = c - g / s_r
                        if ln <= b_r:  # affine piece [c, b_r] holds the root: exact
                            lam[t], done[t] = ln, True
                            continue
                    else:
                        if not math.isfinite(b_r):
                            raise InfeasibleProblemError("a'x = d above the box range")
                        ln = b_r
                else:        # root at or left of c; the leftmost root, as the reference
                    if g == 0.0 and (s_l > 0.0 or not math.isfinite(b_l)):
                        done[t] = True
                        continue
                    hi[t] = c
                    if s_l > 0.0:
                        ln = c - g / s_l
                        if ln >= b_l:
                            lam[t], done[t] = ln, True
                            continue
                    else:
                        if not math.isfinite(b_l):
                            raise InfeasibleProblemError("a'x = d below the box range")
                        ln = b_l
                if not (lo[t] < ln < hi[t]) and math.isfinite(lo[t]) and math.isfinite(hi[t]):
                    ln = 0.5 * (lo[t] + hi[t])
                lam[t] = ln
        self.base.proj_local(A, box, T, lam, 1, self.rec, B=B, coefs=coefs, x_out=x_out,
                             free_out=free_out, ref=ref, base=base, base_lam=base_lam)
        rec = self._fold(self.rec, T, 1)
        host = np.zeros(T, dtype=_lib.PROJ_STATE_DTYPE)
        for t in range(T):
            host[t]["lam"] = lam[t]
            host[t]["sum_v2"], host[t]["sum_r2"], host[t]["sum_dref2"] = rec[t, 0:3]
            if base is not None:  # slot 0 carries the Bregman term (dist.cu)
                host[t]["sum_bh"], host[t]["sum_v2"] = rec[t, 0], 0.0
            host[t]["sum_a2_free"] = rec[t, 3]
            host[t]["nfree"] = int(round(rec[t, 4]))
            host[t]["sum_xv"] = rec[t, 5]
            host[t]["status"] = _lib.PROJ_APPLIED
            host[t]["passes"] = npass
        states[:T].copy_(torch.from_numpy(host.view(np.uint8).reshape(T, -1)))


class ShardedEngine(_Engine):
    """solver._Engine over a rank slice; the Newton system is assembled from the
    rank-summed factor-space Gram."""

    def __init__(self, problem, t_max=4):
        super().__init__(problem, t_max)
        be = self.be
        c2 = be.zeros(1)
        be.dots([(problem.c, None)], c2)
        self.c_norm = math.sqrt(float(c2[0]))
        self.zero = be.zeros(1)
        self.am = be.empty(self.n)

    def gradient(self, g2=None):
        """Unfused: X^T s is all-gathered between the two products."""
        op, be = self.op, self.be
        be.vec(3, 0.0, self.w, self.xp, None, self.s)
        op.xt([self.s], self.gr[:1])
        op.x(self.gr[:1], self.grad.view(1, -1), k=1)
        if g2 is not None:
            be.dots([(self.grad, None)], g2)

    def direction(self, p, sigma, asa=0.0):
        if p == 0:
            return super().direction(p, sigma, asa)
        if self.op.kind == "csr":
            return self._direction_cg(p, sigma, asa)
        be, base, op = self.be, self.be.base, self.op
        if self.q > self.pb_direct_limit():
            raise InternalError("q x q system larger than direct_solve_threshold")
        base.compact(self.free, self.J, self.pcount)
        # M_r = I + X_Jr^T X_Jr (sigma = 1, no rank-one term), summed over ranks
        base.dense_gram(op, self.J, self.pcount, self.n, self.box.a_dev, 1.0, self.zero, self.M,
                        self.m1)
        be.allsum(self.M)
        # u = X_J^T a_J (global), then M = I + sigma (G - u u'/a'a), G = sum M_r - world I
        base.hs_apply_coef(self.free, self.box.a_dev, self.box.a_dev, 1.0, None, 0.0, 0.0, self.am)
        op.xt([self.am], self.gr[1:2])
        base.qspace_assemble(self.q, self.gr[1], asa, sigma, float(be.comm.world), self.M)
        base.chol_solve(self.M, self.q, self.gr[0], -1.0, self.t[0], self.info)
        op.x(self.t, self.qdir.view(1, -1), k=1)
        # d = -s - sigma P_J(Qd) with the global coefficient a_J'(Qd)_J / a_J'a_J
        be.dots([(self.box.a_dev, self.qdir)], self.scal[8:9], mask=self.free)
        aq = float(self.scal[8])
        coef = aq / asa if asa != 0.0 else 0.0
        base.hs_apply_coef(self.free, self.box.a_dev, self.qdir, -sigma, self.s, -1.0, coef,
                           self.dir)
        be.dots([(self.grad, self.dir), (self.w, self.qw), (self.w, self.qdir)], self.scal)
        be.dots([(self.t[0], None)], self.scal[3:4], replicated=True)


    # ------------------------------------------------------------ sparse operator
    CG_BATCH = 16        # iterations between true-residual checks (csrc/driver.cu)
    SPARSE_CG_ETA = 1e-2  # forcing-term cap of the matrix-free route (= the reference's eta)

    def _cg_buffers(self):
        if getattr(self, "_cgq", None) is None:
            e = self.be.empty
            self._cgq = {k: e(self.q) for k in ("u", "uu", "dinv", "y", "r", "z", "pv", "gq",
                                                 "tq")}
            self._cgn = {k: e(self.n) for k in ("zn", "wn")}
        return self._cgq, self._cgn

    def _gram_apply(self, v, out):
        """out = X_J^T X_J v (global q-vector; the rank-one term is applied by the
        caller): X v and the free-row mask are rank-local, X^T is all-gathered."""
        base, op = self.be.base, self.op
        _, nb = self._cg_buffers()
        op.x(v.view(1, -1), nb["zn"].view(1, -1), k=1)
        base.hs_apply_coef(self.free, self.box.a_dev, nb["zn"], 1.0, None, 0.0, 0.0, nb["wn"])
        op.xt([nb["wn"]], out.view(1, -1))

    def _direction_cg(self, p, sigma, asa):
        """Factor-space Jacobi-preconditioned CG of csrc/driver.cu cg_direction_q over row
        shards: (I_q + sigma X_J^T P_J X_J) t = -X^T s.  The q-vectors are replicated
        (every X^T product is rank-summed in rank order), so the CG scalars are the same
        on every rank; one all-gather of a q-vector per iteration.  Stopping test on the
        TRUE Newton residual sigma X X_J^T P X_J r every CG_BATCH iterations against
        min(eta, ||grad||^(1+tau)) (ref solver.py:229, eta capped as the driver)."""
        be, base, op = self.be, self.be.base, self.op
        qb, nb = self._cg_buffers()
        inv_asa = 1.0 / asa if asa != 0.0 else 0.0
        # u = X_J^T a_J; Jacobi dinv = 1 / (1 + sigma max(colsq_J - u^2/a'a, 0))
        base.hs_apply_coef(self.free, self.box.a_dev, self.box.a_dev, 1.0, None, 0.0, 0.0,
                           self.am)
        op.xt([self.am], qb["u"].view(1, -1))
        be.csr_colsq(op, self.free, qb["z"])
        base.vec(5, 0.0, qb["u"], qb["u"], None, qb["uu"])
        base.vec(4, inv_asa, qb["uu"], None, None, qb["uu"])
        base.vec(6, sigma, qb["z"], qb["uu"], None, qb["dinv"])
        # y = 0, r = b = -X^T s, z = D^-1 r, pv = z
        base.vec(4, 0.0, qb["u"], None, None, qb["y"])
        base.vec(4, -1.0, self.gr[0], None, None, qb["r"])
        base.vec(5, 0.0, qb["dinv"], qb["r"], None, qb["z"])
        qb["pv"].copy_(qb["z"])
        be.dots([(qb["r"], qb["z"]), (qb["r"], None)], self.scal[8:10], replicated=True)
        be.dots([(self.grad, None)], self.scal[11:12])
        sc, _ = self.fetch()
        rz, rr = float(sc[8]), float(sc[9])
        gnorm = math.sqrt(max(float(sc[11]), 0.0))
        tol = min(min(self.cg_eta, self.SPARSE_CG_ETA), gnorm ** (1.0 + self.cg_tau))
        done = rr == 0.0
        it = 0
        max_it = 4 * self.cg_max_iters
        while not done and it < max_it:
            for _ in range(self.CG_BATCH):
                if it >= max_it:
                    break
                it += 1
                self._gram_apply(qb["pv"], qb["gq"])
                be.dots([(qb["pv"], None), (qb["pv"], qb["gq"]), (qb["u"], qb["pv"])],
                        self.scal[8:11], replicated=True)
                sc, _ = self.fetch()
                c = float(sc[10]) * inv_asa
                pap = float(sc[8]) + sigma * (float(sc[9]) - c * float(sc[10]))
                alpha = rz / pap if pap > 0.0 else 0.0
                base.vec(2, alpha, qb["y"], qb["pv"], None, qb["y"])
                # r -= alpha (pv + sigma (gq - c u))
                base.vec(2, -alpha, qb["r"], qb["pv"], None, qb["r"])
                base.vec(2, -alpha * sigma, qb["r"], qb["gq"], None, qb["r"])
                base.vec(2, alpha * sigma * c, qb["r"], qb["u"], None, qb["r"])
                base.vec(5, 0.0, qb["dinv"], qb["r"], None, qb["z"])
                be.dots([(qb["r"], qb["z"]), (qb["r"], None)], self.scal[8:10], replicated=True)
                sc, _ = self.fetch()
                rz_new = float(sc[8])
                beta = rz_new / rz if rz != 0.0 else 0.0
                rz = rz_new
                base.vec(2, beta, qb["z"], qb["pv"], None, qb["pv"])
            # true Newton residual: sigma X (X_J^T P X_J r)
            self._gram_apply(qb["r"], qb["gq"])
            be.dots([(qb["u"], qb["r"])], self.scal[8:9], replicated=True)
            sc, _ = self.fetch()
            base.vec(2, -float(sc[8]) * inv_asa, qb["gq"], qb["u"], None, qb["tq"])
            op.x(qb["tq"].view(1, -1), nb["zn"].view(1, -1), k=1)
            be.dots([(nb["zn"], None)], self.scal[8:9])
            sc, _ = self.fetch()
            done = sigma * math.sqrt(max(float(sc[8]), 0.0)) <= tol
        self.counters["cg_iters"] = self.counters.get("cg_iters", 0) + it
        self.t[0].copy_(qb["y"])
        # d = -s - sigma P_J(X t) with the global coefficient a_J'(X t)_J / a_J'a_J
        op.x(self.t, self.qdir.view(1, -1), k=1)
        be.dots([(self.box.a_dev, self.qdir)], self.scal[8:9], mask=self.free)
        sc, _ = self.fetch()
        coef = float(sc[8]) * inv_asa
        base.hs_apply_coef(self.free, self.box.a_dev, self.qdir, -sigma, self.s, -1.0, coef,
                           self.dir)
        # inexact t: the exact image Qd = X (X^T d) keeps Qw = Q w (as the driver)
        op.xt([self.dir], self.gr[1:2])
        op.x(self.gr[1:2], self.qdir.view(1, -1), k=1)
        be.dots([(self.grad, self.dir), (self.w, self.qw), (self.w, self.qdir)], self.scal)
        be.dots([(self.gr[1], None)], self.scal[3:4], replicated=True)


class ShardedQpProblem(QpProblem):
    """Rank slice of min 1/2 x'Qx + c'x s.t. a'x = d, l <= x <= u."""

    def __init__(self, q_op, c, constraint, d_global, comm, layout):
        super().__init__(q_op, c, constraint)
        constraint.d_global = float(d_global)
        self.comm = comm
        self.layout = layout  # (kind, n_phys_total, lo, hi)

    def engine(self):
        if self._engine is None:
            self._engine = ShardedEngine(self)
        return self._engine


def _local_backend(comm, backend=None):
    return ShardedBackend(backend or default_backend(), comm)


def build_csvc_dual_sharded(features, labels, C, comm, backend=None):
    """Rank slice of the C-SVC dual (ref svm.py:95-108): ``features``/``labels`` are
    THIS rank's rows (shard_range gives the conventional split)."""
    be = _local_backend(comm, backend)
    y = np.asarray(labels.detach().cpu().numpy() if isinstance(labels, torch.Tensor) else labels,
                   dtype=np.float64)
    if not np.all(np.abs(y) == 1.0):
        raise InputError("classification labels must be +1/-1")
    if not C > 0:
        raise InputError("C must be positive")
    n_loc = y.shape[0]
    sizes = comm.all_gather_objects(n_loc)
    from .svm import _is_sparse

    if _is_sparse(features):  # CSR rows of this shard (BASELINE configs 3, 4)
        from .operators import CsrKernelOperator

        op = CsrKernelOperator(features, labels=y, backend=be)
    else:
        op = LinearKernelOperator(features, labels=y, backend=be)
    box = BoxLineSet(a=y, d=0.0, l=0.0, u=float(C), backend=be)
    lo = int(sum(sizes[: comm.rank]))
    return ShardedQpProblem(op, -np.ones(n_loc), box, 0.0, comm,
                            ("csvc", int(sum(sizes)), lo, lo + n_loc))


def build_svr_dual_sharded(features, targets, C, epsilon, comm, backend=None):
    """Rank slice of the eps-SVR dual (ref svm.py:111-127): local variables are
    [x+ ; x-] of this rank's rows."""
    be = _local_backend(comm, backend)
    t = np.asarray(targets.detach().cpu().numpy() if isinstance(targets, torch.Tensor) else targets,
                   dtype=np.float64)
    if not C > 0 or epsilon < 0:
        raise InputError("need C > 0 and epsilon >= 0")
    n_loc = t.shape[0]
    sizes = comm.all_gather_objects(n_loc)
    op = LinearKernelOperator(features, svr_block=True, backend=be)
    c = np.concatenate([epsilon - t, epsilon + t])
    a = np.concatenate([np.ones(n_loc), -np.ones(n_loc)])
    box = BoxLineSet(a=a, d=0.0, l=0.0, u=float(C), backend=be)
    lo = int(sum(sizes[: comm.rank]))
    return ShardedQpProblem(op, c, box, 0.0, comm, ("svr", int(sum(sizes)), lo, lo + n_loc))


def solve_loopback(problems, alm_opts=None, ssn_opts=None, device=None):
    """Run the native sharded driver over ``len(problems)`` ranks as host threads of
    this process on ONE GPU (ssnal_loopback_comm_create): ``problems[r]`` is rank r's
    slice, built with the single-GPU builders (``build_csvc_dual`` / ``build_svr_dual``
    on its rows; a nonzero global right-hand side goes in ``constraint.d_global``).
    Each rank runs on its own stream; a collective drains the caller's stream, meets
    the other ranks at a host barrier and sums their buffers in rank order -- no
    kernel waits on another rank, the ranks' kernels only share the GPU.  Returns the
    per-rank SolveReports (x_opt = the rank's slice)."""
    from .solver import AlmOptions, SsnOptions, _alm_solve_native

    alm_opts = alm_opts or AlmOptions()
    ssn_opts = ssn_opts or SsnOptions()
    world = len(problems)
    _lib.load()
    group = ctypes.c_void_p()
    _lib.call("ssnal_loopback_group_create", world, ctypes.byref(group))
    comms = []
    try:
        for r in range(world):
            c = _lib.Comm()
            _lib.call("ssnal_loopback_comm_create", group, r, ctypes.byref(c))
            comms.append(c)
        dev = torch.cuda.current_device() if device is None else device
        out, errs = [None] * world, [None] * world

        def run(r):
            try:
                torch.cuda.set_device(dev)
                with torch.cuda.stream(torch.cuda.Stream(dev)):
                    out[r] = _alm_solve_native(problems[r], alm_opts, ssn_opts, None, None, None,
                                               False, comm=comms[r])
                    torch.cuda.current_stream(dev).synchronize()
            except BaseException as e:  # noqa: BLE001 -- re-raised below
                errs[r] = e

        threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        for e in errs:
            if e is not None:
                raise e
        return out
    finally:
        lib = _lib.load()
        for c in comms:
            lib.ssnal_comm_destroy(ctypes.byref(c))
        lib.ssnal_loopback_group_destroy(group)


def gather_solution(problem, x_local):
    """Full dual vector (reference ordering) on every rank, from the rank slices."""
    comm = problem.comm
    x = torch.as_tensor(x_local, dtype=F64).cpu()
    parts = comm.all_gather_objects(x.numpy())
    kind = problem.layout[0]
    if kind == "csvc":
        return np.concatenate(parts)
    plus = np.concatenate([p[: p.size // 2] for p in parts])
    minus = np.concatenate([p[p.size // 2:] for p in parts])
    return np.concatenate([plus, minus])


__all__ = ["ShardComm", "ShardedBackend", "ShardedEngine", "ShardedQpProblem", "shard_range",
           "build_csvc_dual_sharded", "build_svr_dual_sharded", "gather_solution",
           "solve_loopback"]
