"""Implicit Q operators in factor form Q = X X^T (device resident).

ref kernels.py builds Q_ij = y_i y_j K(x_i, x_j) column by column (KernelOperator
:68-154), the SVR block [[K,-K],[-K,K]] (BlockKernelOperator :181-215) and an
explicit matrix (DenseOperator :218-238).  For the linear kernel all three are
Q = X X^T with

    C-SVC  X = diag(y) A          (LinearKernelOperator(A, labels=y))
    SVR    X = [A; -A]            (LinearKernelOperator(A, svr_block=True))
    dense  X = V diag(sqrt(ev+))  (DenseOperator(Q): host eigendecomposition once)

so the hot path only ever streams A (csrc/dense.cu) and never forms an n x n
block.  ``matvec`` / ``columns`` / ``submatrix`` / ``diag`` keep the reference
operator protocol for callers.
"""

import numpy as np
import torch

from .backend import F64, as_device, check_vector, default_backend
from .errors import InputError


class LinearKernelOperator:
    """Q = X X^T, X = S diag(labels) A, A row-major n x q (fp64, on the device)."""

    kind = "dense"

    def __init__(self, samples, labels=None, svr_block=False, backend=None):
        self.backend = be = backend or default_backend()
        A = as_device(samples, be)
        if A.dim() != 2:
            raise InputError("samples must be an n x q matrix")
        self.A = A
        self.n_phys, self.q = A.shape
        self.lda = A.stride(0)
        self.svr_block = bool(svr_block)
        self.n = 2 * self.n_phys if self.svr_block else self.n_phys
        if labels is not None:
            if isinstance(labels, torch.Tensor) and labels.is_cuda:
                lab = as_device(labels, be)
                check_vector(lab, self.n_phys, "labels")
                if not bool(torch.all(lab.abs() == 1.0)):
                    raise InputError("labels must be +1/-1")
            else:  # host labels: validated on the host (no device round trip)
                lab_h = np.asarray(labels.numpy() if isinstance(labels, torch.Tensor) else labels,
                                   dtype=np.float64)
                if lab_h.ndim != 1 or lab_h.shape[0] != self.n_phys:
                    raise InputError(f"labels: expected a vector of length {self.n_phys}")
                if not np.all(np.abs(lab_h) == 1.0):
                    raise InputError("labels must be +1/-1")
                lab = as_device(lab_h, be)
            self.row_sign = lab
        else:
            self.row_sign = None

    # -- factor products (device, async) -------------------------------------
    def xt(self, vs, out=None):
        """X^T [v_0 .. v_{k-1}] -> q x k column-major buffer (returned as (k, q))."""
        out = out if out is not None else self.backend.empty((len(vs), self.q))
        self.backend.dense_xt(self, vs, out)
        return out

    def x(self, d, out=None, k=1):
        """X d for d a (k, q) buffer -> (k, n) buffer."""
        out = out if out is not None else self.backend.empty((k, self.n))
        self.backend.dense_x(self, d, out, k)
        return out

    # -- reference operator protocol -------------------------------------------
    def matvec(self, v):
        v = as_device(v, self.backend)
        check_vector(v, self.n, "matvec")
        return self.x(self.xt([v]))[0]

    def _rows(self, idx):
        idx = torch.as_tensor(idx, dtype=torch.long, device=self.A.device)
        if idx.numel() and (int(idx.min()) < 0 or int(idx.max()) >= self.n):
            raise InputError("column index out of range")
        phys = idx % self.n_phys
        rows = self.A[phys]
        sgn = torch.ones(idx.numel(), dtype=F64, device=self.A.device)
        if self.row_sign is not None:
            sgn = sgn * self.row_sign[phys]
        if self.svr_block:
            sgn = torch.where(idx >= self.n_phys, -sgn, sgn)
        return rows, sgn

    def columns(self, idx):
        """Dense n x p block Q[:, idx] (for callers; not on the hot path)."""
        rows, sgn = self._rows(idx)
        d = (rows * sgn[:, None]).contiguous()  # (p, q) == columns of X^T
        out = self.backend.empty((d.shape[0], self.n))
        for j in range(0, d.shape[0], 2):
            k = min(2, d.shape[0] - j)
            self.backend.dense_x(self, d[j:j + k], out[j:j + k], k)
        return out.T

    def submatrix(self, idx):
        rows, sgn = self._rows(idx)
        r = rows * sgn[:, None]
        return r @ r.T

    def diag(self):
        d = (self.A * self.A).sum(dim=1)
        return torch.cat([d, d]) if self.svr_block else d


class CsrKernelOperator:
    """Q = X X^T for sparse samples: X = diag(labels) A, A in CSR (device), with a CSC
    copy and a segment plan for the deterministic balanced transposed product,
    built once here on the host (numpy/scipy, not on the solve path)."""

    kind = "csr"
    SEG = 2048  # max nonzeros per warp segment of the CSC product
    HOT_MAX = 4096        # SSNAL_CSR_HOT_MAX: columns staged in shared memory (32 KB of d)
    HOT_MIN_SHARE = 0.25  # staging pays when the hot columns hold at least this share of nnz

    def __init__(self, samples, labels=None, backend=None):
        import ctypes

        import scipy.sparse as sp

        from . import _lib

        self.backend = be = backend or default_backend()
        if isinstance(samples, tuple):
            indptr, indices, data, shape = samples
            A = sp.csr_matrix((data, indices, indptr), shape=shape)
        else:
            A = sp.csr_matrix(samples)
        A.sum_duplicates()  # sorted, duplicate-free rows (the Gram merges rely on it)
        A = A.astype(np.float64)
        self.n_phys, self.q = A.shape
        self.n = self.n_phys
        self.nnz = int(A.nnz)
        self.svr_block = False
        self.lda = self.q
        C = A.tocsc()
        C.sort_indices()
        colptr = C.indptr.astype(np.int64)
        lens = np.diff(colptr)
        nseg_col = np.maximum(1, -(-lens // self.SEG))
        seg_col = np.repeat(np.arange(self.q, dtype=np.int64), nseg_col)
        first = np.repeat(np.cumsum(nseg_col) - nseg_col, nseg_col)
        k = np.arange(seg_col.size) - first
        seg_beg = colptr[seg_col] + k * self.SEG
        seg_end = np.minimum(seg_beg + self.SEG, colptr[seg_col + 1])
        split = nseg_col[seg_col] > 1
        seg_slot = np.full(seg_col.size, -1, dtype=np.int64)
        seg_slot[split] = np.arange(int(split.sum()))
        fold_cols = np.flatnonzero(nseg_col > 1)
        fold_beg = np.concatenate([[0], np.cumsum(nseg_col[fold_cols])]).astype(np.int32)
        # hot-column staging of the CG's X_J d (csrc/sparse.cu csrj_xd_dot_hot_kernel): when
        # the HOT_MAX most populated columns hold a sizeable share of the entries (Zipf
        # popularity), their d entries are served from shared memory
        nhot = int(min(self.HOT_MAX, self.q))
        order = np.argsort(-lens, kind="stable")[:nhot]
        if self.nnz == 0 or lens[order].sum() < self.HOT_MIN_SHARE * self.nnz:
            nhot, order = 0, order[:0]
        hot_rank = np.full(self.q, -1, dtype=np.int32)
        hot_rank[order] = np.arange(nhot, dtype=np.int32)
        self.nhot = nhot
        from .backend import H2D

        def dev(a, dt):
            t = torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=be.device)
            if be.device.type == "cuda":
                H2D["bytes"] += t.numel() * t.element_size()
            return t

        self._t = {
            "indptr": dev(A.indptr.astype(np.int64), torch.int64),
            "indices": dev(A.indices.astype(np.int32), torch.int32),
            "values": dev(A.data, torch.float64),
            "colptr": dev(colptr, torch.int64),
            "rowidx": dev(C.indices.astype(np.int32), torch.int32),
            "valt": dev(C.data, torch.float64),
            "seg_beg": dev(seg_beg, torch.int64), "seg_end": dev(seg_end, torch.int64),
            "seg_col": dev(seg_col.astype(np.int32), torch.int32),
            "seg_slot": dev(seg_slot.astype(np.int32), torch.int32),
            "fold_col": dev(fold_cols.astype(np.int32) if fold_cols.size else np.zeros(1, np.int32),
                            torch.int32),
            "fold_beg": dev(fold_beg if fold_cols.size else np.zeros(2, np.int32), torch.int32),
            "hot_cols": dev(order.astype(np.int32) if nhot else np.zeros(1, np.int32), torch.int32),
            "hot_rank": dev(hot_rank, torch.int32),
        }
        if labels is not None:
            if isinstance(labels, torch.Tensor) and labels.is_cuda:
                lab = as_device(labels, be)
                check_vector(lab, self.n_phys, "labels")
                if not bool(torch.all(lab.abs() == 1.0)):
                    raise InputError("labels must be +1/-1")
            else:  # host labels: validated on the host (no device round trip)
                lab_h = np.asarray(labels.numpy() if isinstance(labels, torch.Tensor) else labels,
                                   dtype=np.float64)
                if lab_h.ndim != 1 or lab_h.shape[0] != self.n_phys:
                    raise InputError(f"labels: expected a vector of length {self.n_phys}")
                if not np.all(np.abs(lab_h) == 1.0):
                    raise InputError("labels must be +1/-1")
                lab = as_device(lab_h, be)
            self.row_sign = lab
        else:
            self.row_sign = None
        self.nslots = int(split.sum())
        self.part = be.zeros(max(self.nslots, 1))
        p = lambda name: self._t[name].data_ptr()  # noqa: E731
        self.c_op = _lib.CsrOperator(
            n=self.n, q=self.q, nnz=self.nnz, indptr=p("indptr"), indices=p("indices"),
            values=p("values"), colptr=p("colptr"), rowidx=p("rowidx"), valt=p("valt"),
            row_sign=None if self.row_sign is None else self.row_sign.data_ptr(),
            nseg=int(seg_col.size), seg_beg=p("seg_beg"), seg_end=p("seg_end"),
            seg_col=p("seg_col"), seg_slot=p("seg_slot"), nfold=int(fold_cols.size),
            fold_col=p("fold_col"), fold_beg=p("fold_beg"), nslots=self.nslots,
            nhot=nhot, hot_cols=p("hot_cols"), hot_rank=p("hot_rank"))
        self._cref = ctypes.byref(self.c_op)
        self.host_csr = A  # kept for callers (oracle checks, columns())

    def xt(self, vs, out=None):
        """X^T v_j on the CSC plan (through the backend, so a sharded backend can sum
        the rank partials)."""
        out = out if out is not None else self.backend.empty((len(vs), self.q))
        for j, v in enumerate(vs):
            self.backend.csr_xt(self, v, out[j])
        return out

    def x(self, d, out=None, k=1):
        out = out if out is not None else self.backend.empty((k, self.n))
        for j in range(k):
            self.backend.csr_x(self, d[j], out[j])
        return out

    def matvec(self, v):
        v = as_device(v, self.backend)
        check_vector(v, self.n, "matvec")
        return self.x(self.xt([v]))[0]

    def diag(self):
        a = self.host_csr
        return torch.as_tensor(np.asarray(a.multiply(a).sum(axis=1)).ravel(),
                               device=self.backend.device)


class DenseOperator(LinearKernelOperator):
    """Explicit symmetric PSD Q (ref kernels.py:218-238), factored once on the host
    as Q = X X^T with X = V diag(sqrt(max(ev, 0)))."""

    def __init__(self, q, backend=None):
        qh = np.asarray(q.detach().cpu().numpy() if isinstance(q, torch.Tensor) else q,
                        dtype=np.float64)
        if qh.ndim != 2 or qh.shape[0] != qh.shape[1]:
            raise InputError("Q must be square")
        ev, vec = np.linalg.eigh(0.5 * (qh + qh.T))
        keep = ev > 1e-13 * max(float(ev.max()), 1.0)
        factor = vec[:, keep] * np.sqrt(ev[keep])[None, :]
        if factor.shape[1] == 0:
            factor = np.zeros((qh.shape[0], 1))
        super().__init__(np.ascontiguousarray(factor), backend=backend)
        self.q_host = qh
