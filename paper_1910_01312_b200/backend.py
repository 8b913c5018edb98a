"""CUDA backend: thin typed wrappers over the C-ABI, operating on torch tensors.

torch supplies device memory and the current stream only; every arithmetic
operation of the SSsNAL path runs in the sm_100a library.  All calls are
asynchronous on torch's current stream; ``fetch_*`` helpers are the only
host synchronisation points.
"""

import numpy as np
import torch

from . import _lib
from .errors import CudaUnavailableError, InputError

F64 = torch.float64


def _ptr(t):
    return None if t is None else t.data_ptr()


class CudaBackend:
    """One per device.  Owns no problem-sized buffers (see solver.Workspace)."""

    name = "cuda"

    def __init__(self, device=None):
        if not torch.cuda.is_available():
            raise CudaUnavailableError("no CUDA device visible (there is no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        self.lib = _lib.load()
        _lib.call("ssnal_device_check", self.device.index)
        self._ws = {}
        self.timing = None  # list of (op, start_event, end_event, algorithmic bytes) when on

    # ---------------------------------------------------------------- profiling
    def start_timing(self):
        self.timing = []

    def stop_timing(self):
        """Per-op totals {op: (launch count, seconds, algorithmic bytes)} from CUDA events
        recorded on the launching stream around every timed op."""
        torch.cuda.synchronize(self.device)
        out = {}
        for op, e0, e1, nbytes in self.timing or []:
            c, t, b = out.get(op, (0, 0.0, 0.0))
            out[op] = (c + 1, t + e0.elapsed_time(e1) * 1e-3, b + nbytes)
        self.timing = None
        return out

    def _timed(self, op, nbytes, fn, *args):
        if self.timing is None:
            return fn(*args)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        s = torch.cuda.current_stream(self.device)
        e0.record(s)
        fn(*args)
        e1.record(s)
        self.timing.append((op, e0, e1, nbytes))

    def launch_count(self):
        return int(self.lib.ssnal_launch_count())

    # ---------------------------------------------------------------- memory
    def empty(self, shape, dtype=F64):
        return torch.empty(shape, dtype=dtype, device=self.device)

    def zeros(self, shape, dtype=F64):
        return torch.zeros(shape, dtype=dtype, device=self.device)

    def ws(self, key, nbytes):
        """Zero-initialised scratch (tickets inside must start at 0), grown on demand."""
        buf = self._ws.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.zeros(max(int(nbytes), 256), dtype=torch.uint8, device=self.device)
            self._ws[key] = buf
        return buf

    def stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def synchronize(self):
        torch.cuda.current_stream(self.device).synchronize()

    @staticmethod
    def host_buffer(shape, dtype):
        return torch.empty(shape, dtype=dtype, pin_memory=True)

    def new_states(self, T):
        return torch.zeros((T, _lib.PROJ_STATE_DTYPE.itemsize), dtype=torch.uint8,
                           device=self.device)

    @staticmethod
    def read_states(states_host):
        return states_host.numpy().view(_lib.PROJ_STATE_DTYPE).reshape(-1)

    # ---------------------------------------------------------------- projection
    # default search: this many warm-started Newton passes, then K-ary passes take over
    NEWTON_PASSES = 3
    KARY_PASSES = 0

    def project(self, A, box, states, T=1, B=None, coefs=None, x_out=None, free_out=None,
                ref=None, phases=None, passes=None, hint=0.0, newton=None, base=None,
                base_lam=0.0):
        n = box.n
        if newton is None:
            newton = self.NEWTON_PASSES
        if passes is None:
            passes = self.KARY_PASSES
        if phases is None:  # Newton ends exactly; the K-ary exact phase only in fallbacks
            phases = _lib.PHASE_APPLY if newton > 0 else 7
        coef_arr = None
        if B is not None:
            coef_arr = (_lib.ctypes.c_double * T)(*[float(c) for c in coefs])
        ws = self.ws("proj", self.lib.ssnal_project_ws_bytes(n, T))
        # per streaming launch: v (+ B) and a, (+ l, u vectors)
        per_phase = 8 * n * (2 + (B is not None) + (box.l_dev is not None) + (box.u_dev is not None))
        self._timed(
            "project", per_phase * (newton + 1), _lib.call,
            "ssnal_project_ex", _ptr(A), _ptr(B),
            _lib.ctypes.cast(coef_arr, _lib.ctypes.c_void_p) if coef_arr is not None else None,
            _ptr(box.a_dev), _ptr(box.l_dev), _ptr(box.u_dev), box.l_const, box.u_const, box.d,
            n, T, _ptr(states), _ptr(ws), _ptr(x_out), _ptr(free_out), _ptr(ref), _ptr(base),
            float(base_lam), float(hint), int(newton), phases, passes, self.stream())

    def project_sync(self, A, box, states, T=1, B=None, coefs=None, x_out=None, free_out=None,
                     ref=None, hint=0.0):
        """Project and return the host copy of the T state records (one sync,
        plus a rare extra round if a trial needed more bracketing passes)."""
        self.project(A, box, states, T, B, coefs, x_out, free_out, ref, hint=hint)
        st = self.read_states(states[:T].cpu())
        extra = 0
        while np.any((st["status"] >= 0) & (st["status"] != _lib.PROJ_APPLIED)):
            extra += 1
            if extra > 20:
                raise RuntimeError("projection failed to bracket the multiplier")
            self.project(A, box, states, T, B, coefs, x_out, free_out, ref,
                         phases=_lib.PHASE_EXACT | _lib.PHASE_APPLY, passes=8, newton=0)
            st = self.read_states(states[:T].cpu())
        return st

    # ---------------------------------------------------------------- vectors
    def dots(self, pairs, out, mask=None):
        """out[j] = sum m x_j y_j (y None => x^2); pairs <= 8; async."""
        k = len(pairs)
        n = pairs[0][0].numel()
        if any(x.numel() != n or (y is not None and y.numel() != n) for x, y in pairs):
            raise InputError("dots: all vectors of one call must have the same length")
        xs, keep1 = _lib.ptr_array([_ptr(x) for x, _ in pairs])
        ys, keep2 = _lib.ptr_array([_ptr(y) for _, y in pairs])
        ws = self.ws("reduce", self.lib.ssnal_reduce_ws_bytes(n, k))
        _lib.call("ssnal_dots", k, xs, ys, _ptr(mask), n, _ptr(out), _ptr(ws), self.stream())
        del keep1, keep2

    def vec(self, op, alpha, x, y, z, out):
        _lib.call("ssnal_vec", op, x.numel(), float(alpha), _ptr(x), _ptr(y), _ptr(z),
                  _ptr(out), self.stream())

    def hs_apply(self, free, a, y, beta, add, alpha, out):
        n = y.numel()
        ws = self.ws("hs", self.lib.ssnal_reduce_ws_bytes(n, 2))
        _lib.call("ssnal_hs_apply", _ptr(free), _ptr(a), _ptr(y), n, float(beta), _ptr(add),
                  float(alpha), _ptr(out), _ptr(ws), self.stream())

    def compact(self, mask, idx_out, count_out):
        n = mask.numel()
        ws = self.ws("compact", self.lib.ssnal_compact_ws_bytes(n))
        _lib.call("ssnal_compact", _ptr(mask), n, _ptr(idx_out), _ptr(count_out), _ptr(ws),
                  self.stream())

    # ---------------------------------------------------------------- dense operator
    @staticmethod
    def dense_bytes(op, k, direction):
        """Algorithmic HBM bytes of one X^T V (direction 't') or X D ('x') product:
        the sample matrix once, the row signs, the k input and k output vectors."""
        a_bytes = 8 * op.n_phys * op.q + (8 * op.n_phys if op.row_sign is not None else 0)
        if direction == "t":
            return a_bytes + 8 * k * op.n + 8 * k * op.q
        return a_bytes + 8 * k * op.q + 8 * k * op.n

    def dense_xt(self, op, vs, out):
        k = len(vs)
        arr, keep = _lib.ptr_array([_ptr(v) for v in vs])
        ws = self.ws("xt", self.lib.ssnal_dense_xt_ws_bytes(op.n_phys, op.q, k))
        self._timed("dense_xt", self.dense_bytes(op, k, "t"), _lib.call, "ssnal_dense_xt",
                    _ptr(op.A), op.n_phys, op.q, op.lda, _ptr(op.row_sign), int(op.svr_block), k,
                    arr, _ptr(out), _ptr(ws), self.stream())
        del keep

    def dense_x(self, op, d, out, k=1):
        self._timed("dense_x", self.dense_bytes(op, k, "x"), _lib.call, "ssnal_dense_x",
                    _ptr(op.A), op.n_phys, op.q, op.lda, _ptr(op.row_sign), int(op.svr_block), k,
                    _ptr(d), _ptr(out), self.stream())

    def dense_gradient(self, op, w, xp, s_out, g_r, grad, g2):
        """s = w - xp, g_r = X^T s, grad = X g_r, g2 = ||grad||^2 (device), fused."""
        ws = self.ws("gradient", self.lib.ssnal_gradient_ws_bytes(op.n_phys, op.q))
        self._timed("dense_gradient", 2 * self.dense_bytes(op, 1, "t"), _lib.call,
                    "ssnal_dense_gradient", _ptr(op.A), op.n_phys, op.q, op.lda, _ptr(op.row_sign),
                    int(op.svr_block), _ptr(w), _ptr(xp), _ptr(s_out), _ptr(g_r), _ptr(grad),
                    _ptr(g2), _ptr(ws), self.stream())

    def direction_epilogue(self, op, t, qdir, free, a, asa_dev, s, sigma, grad, w, qw, dir_out,
                           dots4):
        """qdir = X t, dir = -s - sigma P(qdir), dots4 = {g'dir, w'qw, w'qdir, t't} (fused)."""
        ws = self.ws("gradient", self.lib.ssnal_gradient_ws_bytes(op.n_phys, op.q))
        self._timed("dense_x", self.dense_bytes(op, 1, "x"), _lib.call,
                    "ssnal_dense_direction_epilogue", _ptr(op.A), op.n_phys, op.q, op.lda,
                    _ptr(op.row_sign), int(op.svr_block), _ptr(t), _ptr(qdir), _ptr(free), _ptr(a),
                    _ptr(asa_dev), _ptr(s), float(sigma), _ptr(grad), _ptr(w), _ptr(qw),
                    _ptr(dir_out), _ptr(dots4), _ptr(ws), self.stream())

    def dense_gram(self, op, J, p_dev, p_max, a, sigma, asa_dev, M, m1):
        ws = self.ws("gram", self.lib.ssnal_gram_ws_bytes(op.q))
        self._timed("dense_gram", 0, _lib.call, "ssnal_dense_gram", _ptr(op.A), op.n_phys, op.q,
                    op.lda, _ptr(op.row_sign), int(op.svr_block), _ptr(J), _ptr(p_dev),
                    int(p_max), _ptr(a), float(sigma), _ptr(asa_dev), _ptr(M), _ptr(m1), _ptr(ws),
                    self.stream())

    def newton_pspace(self, op, J, p, grad, a, sigma, asa, g_r, t, info):
        ws = self.ws("pspace", self.lib.ssnal_pspace_ws_bytes(p, op.q))
        self._timed("newton_pspace", 0, _lib.call, "ssnal_dense_newton_pspace", _ptr(op.A),
                    op.n_phys, op.q, op.lda, _ptr(op.row_sign), int(op.svr_block), _ptr(J), int(p),
                    _ptr(grad), _ptr(a), float(sigma), float(asa), _ptr(g_r), _ptr(t), _ptr(info),
                    _ptr(ws), self.stream())

    def chol_solve(self, M, m, b, scale, x, info):
        self._timed("chol_solve", 16 * m * m, _lib.call, "ssnal_chol_solve", _ptr(M), int(m),
                    _ptr(b), float(scale), _ptr(x), _ptr(info), self.stream())

    # ---------------------------------------------------------------- CSR operator
    def csr_xt(self, op, v, out):
        """out = X^T v (q) on the operator's CSC segment plan."""
        _lib.call("ssnal_csr_xt", op._cref, _ptr(v), _ptr(out), _ptr(op.part), self.stream())

    def csr_x(self, op, d, out):
        """out = X d (n)."""
        _lib.call("ssnal_csr_xd", op._cref, None, op.n, _ptr(d), _ptr(out), self.stream())

    def csr_colsq(self, op, keep, out):
        """out[k] = sum over rows with keep != 0 of A_ik^2 (Jacobi diagonal of X_J^T X_J)."""
        _lib.call("ssnal_csr_colsq", op._cref, _ptr(keep), _ptr(out), _ptr(op.part),
                  self.stream())

    # ---------------------------------------------------------------- sharded path
    def proj_local(self, A, box, T, lam, mode, rec, B=None, coefs=None, x_out=None,
                   free_out=None, ref=None, base=None, base_lam=0.0):
        """Shard-local projection records at host multipliers ``lam`` (csrc/dist.cu)."""
        n = box.n
        lam_arr = (_lib.ctypes.c_double * T)(*[float(v) for v in lam])
        coef_arr = None
        if B is not None:
            coef_arr = (_lib.ctypes.c_double * T)(*[float(c) for c in coefs])
        ws = self.ws("proj_local", self.lib.ssnal_proj_local_ws_bytes(n, T))
        _lib.call("ssnal_proj_local", _ptr(A), _ptr(B),
                  _lib.ctypes.cast(coef_arr, _lib.ctypes.c_void_p) if coef_arr is not None else None,
                  _lib.ctypes.cast(lam_arr, _lib.ctypes.c_void_p), _ptr(box.a_dev), _ptr(box.l_dev),
                  _ptr(box.u_dev), box.l_const, box.u_const, n, T, int(mode), _ptr(x_out),
                  _ptr(free_out), _ptr(ref), _ptr(base), float(base_lam), _ptr(rec), _ptr(ws),
                  self.stream())

    def sum_slices(self, k, src, out):
        """out = sum of the k equal slices of src, in slice order."""
        _lib.call("ssnal_sum_slices", int(k), out.numel(), _ptr(src), _ptr(out), self.stream())

    def hs_apply_coef(self, free, a, y, beta, add, alpha, coef, out):
        _lib.call("ssnal_hs_apply_coef", _ptr(free), _ptr(a), _ptr(y), y.numel(), float(beta),
                  _ptr(add), float(alpha), float(coef), _ptr(out), self.stream())

    def qspace_assemble(self, m, u, asa, sigma, shift, M):
        _lib.call("ssnal_qspace_assemble", int(m), _ptr(u), float(asa), float(sigma), float(shift),
                  _ptr(M), self.stream())


_DEFAULT = {}


def default_backend(device=None):
    key = str(device)
    if key not in _DEFAULT:
        _DEFAULT[key] = CudaBackend(device)
    return _DEFAULT[key]


# host -> device bytes moved by as_device (bench.py's e2e copy declaration reads it)
H2D = {"bytes": 0}


def as_device(x, backend, dtype=F64):
    """Host (numpy / list / CPU tensor) or device tensor -> contiguous device tensor."""
    if isinstance(x, torch.Tensor):
        if x.device.type == "cpu" and backend.device.type == "cuda":
            H2D["bytes"] += x.numel() * torch.empty((), dtype=dtype).element_size()
        t = x.to(device=backend.device, dtype=dtype)
    else:
        arr = np.asarray(x, dtype=np.float64 if dtype == F64 else None)
        if backend.device.type == "cuda":
            H2D["bytes"] += arr.size * torch.empty((), dtype=dtype).element_size()
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(device=backend.device, dtype=dtype)
    if not t.is_contiguous():
        t = t.contiguous()
    return t


def check_vector(v, n, what):
    if v.dim() != 1 or v.numel() != n:
        raise InputError(f"{what}: expected a vector of length {n}, got shape {tuple(v.shape)}")
