"""TEST-ONLY CPU stand-in for CudaBackend (numpy / oracle arithmetic).

It lets the host-side control flow of the solver (solver._Engine, the ALM /
SsN loops, the line search batching, the sharded plumbing) run in the CPU test
suite.  It is injected explicitly by tests; the product package never imports
it and has no CPU path of its own.
"""

import numpy as np
import torch

import oracle as O
from paper_1910_01312_b200 import _lib

F64 = torch.float64



def _bregman(x, base, v, a, lam, base_lam):
    """sum (x - Pi_b)(v - (x + Pi_b)/2 - lam_bar a): the trial's Bregman term
    (csrc/proj.cu bregman_term); 0 without a base point."""
    if base is None:
        return 0.0
    xb = base.numpy()
    return float(((x - xb) * (v - 0.5 * (x + xb) - 0.5 * (lam + base_lam) * a)).sum())

class CpuTestBackend:
    name = "cpu-test"

    def __init__(self):
        self.device = torch.device("cpu")
        self.calls = {}

    def _count(self, k):
        self.calls[k] = self.calls.get(k, 0) + 1

    # memory ------------------------------------------------------------------
    def empty(self, shape, dtype=F64):
        return torch.empty(shape, dtype=dtype)

    def zeros(self, shape, dtype=F64):
        return torch.zeros(shape, dtype=dtype)

    def ws(self, key, nbytes):
        return torch.zeros(max(int(nbytes), 256), dtype=torch.uint8)

    def stream(self):
        return None

    def synchronize(self):
        pass

    @staticmethod
    def host_buffer(shape, dtype):
        return torch.empty(shape, dtype=dtype)

    def new_states(self, T):
        return torch.zeros((T, _lib.PROJ_STATE_DTYPE.itemsize), dtype=torch.uint8)

    @staticmethod
    def read_states(states_host):
        return states_host.numpy().view(_lib.PROJ_STATE_DTYPE).reshape(-1)

    # projection --------------------------------------------------------------
    def project(self, A, box, states, T=1, B=None, coefs=None, x_out=None, free_out=None,
                ref=None, phases=7, passes=6, hint=0.0, newton=3, base=None, base_lam=0.0):
        self._count("project")
        a = box.a_dev.numpy()
        l = box.l.numpy()
        u = box.u.numpy()
        bl = O.BoxLine(a, box.d, l, u)
        rec = self.read_states(states)
        for t in range(T):
            v = A.numpy().copy()
            if B is not None:
                v = v - float(coefs[t]) * B.numpy()
            x, lam, free = O.project(v, bl)
            r = v - x
            rec[t]["lam"] = lam
            rec[t]["sum_v2"] = 0.0 if base is not None else float(v @ v)
            rec[t]["sum_bh"] = _bregman(x, base, v, a, lam, base_lam)
            rec[t]["sum_r2"] = float(r @ r)
            rec[t]["sum_xv"] = float(x @ (2.0 * v - x))
            rec[t]["sum_dref2"] = float(((x - ref.numpy()) ** 2).sum()) if ref is not None else 0.0
            rec[t]["sum_a2_free"] = float((a[free] ** 2).sum())
            rec[t]["nfree"] = int(free.sum())
            rec[t]["status"] = _lib.PROJ_APPLIED
            rec[t]["passes"] = 1
            if x_out is not None:
                x_out.view(-1, box.n)[t].copy_(torch.from_numpy(x))
            if free_out is not None:
                free_out.view(-1, box.n)[t].copy_(torch.from_numpy(free.astype(np.uint8)))

    # vectors -----------------------------------------------------------------
    def dots(self, pairs, out, mask=None):
        self._count("dots")
        m = None if mask is None else mask.numpy().astype(bool)
        for j, (x, y) in enumerate(pairs):
            xv = x.numpy()
            yv = xv if y is None else y.numpy()
            prod = xv * yv
            out[j] = float(prod[m].sum() if m is not None else prod.sum())

    def vec(self, op, alpha, x, y, z, out):
        self._count("vec")
        xv = x.numpy()
        if op == 0:
            r = xv + alpha * (y.numpy() + (z.numpy() if z is not None else 0.0))
        elif op == 1:
            r = (xv - y.numpy()) - z.numpy()
        elif op == 2:
            r = xv + alpha * y.numpy()
        elif op == 3:
            r = xv - y.numpy()
        elif op == 5:
            r = xv * y.numpy()
        elif op == 6:
            r = 1.0 / (1.0 + alpha * np.maximum(xv - y.numpy(), 0.0))
        else:
            r = alpha * xv
        out.copy_(torch.from_numpy(np.ascontiguousarray(r)))

    def hs_apply(self, free, a, y, beta, add, alpha, out):
        self._count("hs_apply")
        py = O.hs_apply(free.numpy().astype(bool), a.numpy(), y.numpy())
        r = beta * py
        if add is not None:
            r = alpha * add.numpy() + r
        out.copy_(torch.from_numpy(r))

    def compact(self, mask, idx_out, count_out):
        self._count("compact")
        idx = np.flatnonzero(mask.numpy())
        idx_out[: idx.size] = torch.from_numpy(idx.astype(np.int32))
        count_out[0] = idx.size

    # CSR operator --------------------------------------------------------------
    @staticmethod
    def _csr_signed(op):
        A = op.host_csr
        if op.row_sign is not None:
            import scipy.sparse as sp
            A = sp.diags(op.row_sign.cpu().numpy()) @ A
        return A.tocsr()

    def csr_xt(self, op, v, out):
        self._count("csr_xt")
        out.copy_(torch.from_numpy(np.ascontiguousarray(self._csr_signed(op).T @ v.numpy())))

    def csr_x(self, op, d, out):
        self._count("csr_x")
        out.copy_(torch.from_numpy(np.ascontiguousarray(self._csr_signed(op) @ d.numpy())))

    def csr_colsq(self, op, keep, out):
        self._count("csr_colsq")
        A = op.host_csr
        k = keep.numpy().astype(np.float64)
        out.copy_(torch.from_numpy(np.ascontiguousarray(A.multiply(A).T @ k)))

    # dense operator ------------------------------------------------------------
    @staticmethod
    def _x_rows(op):
        A = op.A.numpy()
        if op.row_sign is not None:
            A = op.row_sign.numpy()[:, None] * A
        return np.vstack([A, -A]) if op.svr_block else A

    def dense_xt(self, op, vs, out):
        self._count("dense_xt")
        X = self._x_rows(op)
        for j, v in enumerate(vs):
            out[j] = torch.from_numpy(X.T @ v.numpy())

    def dense_x(self, op, d, out, k=1):
        self._count("dense_x")
        X = self._x_rows(op)
        dd = d.reshape(k, -1).numpy()
        o = out.reshape(k, -1)
        for j in range(k):
            o[j] = torch.from_numpy(X @ dd[j])

    def dense_gradient(self, op, w, xp, s_out, g_r, grad, g2):
        self._count("dense_gradient")
        X = self._x_rows(op)
        s = w.numpy() - xp.numpy()
        s_out.copy_(torch.from_numpy(s))
        gr = X.T @ s
        g_r.copy_(torch.from_numpy(gr))
        gv = X @ gr
        grad.copy_(torch.from_numpy(gv))
        g2.view(-1)[0] = float(gv @ gv)

    def direction_epilogue(self, op, t, qdir, free, a, asa_dev, s, sigma, grad, w, qw, dir_out,
                           dots4):
        self._count("direction_epilogue")
        X = self._x_rows(op)
        qd = X @ t.reshape(-1).numpy()
        qdir.view(-1).copy_(torch.from_numpy(qd))
        fm = free.numpy().astype(bool)
        av = a.numpy()
        aa = float(asa_dev.view(-1)[0])
        coef = float((av[fm] * qd[fm]).sum()) / aa if aa != 0.0 else 0.0
        d = -s.numpy() - sigma * np.where(fm, qd - coef * av, 0.0)
        dir_out.copy_(torch.from_numpy(d))
        tv = t.reshape(-1).numpy()
        vals = [float(grad.numpy() @ d), float(w.numpy() @ qw.numpy()), float(w.numpy() @ qd),
                float(tv @ tv)]
        for k in range(4):
            dots4.view(-1)[k] = vals[k]

    def dense_gram(self, op, J, p_dev, p_max, a, sigma, asa_dev, M, m1):
        self._count("dense_gram")
        X = self._x_rows(op)
        p = int(p_dev[0])
        idx = J[:p].numpy().astype(np.int64)
        Z = X[idx]
        G = Z.T @ Z
        m = Z.T @ a.numpy()[idx]
        asa = float(asa_dev[0])
        if asa != 0.0:
            G = G - np.outer(m, m) / asa
        M.copy_(torch.from_numpy(np.eye(G.shape[0]) + sigma * G))
        m1.copy_(torch.from_numpy(m))

    def newton_pspace(self, op, J, p, grad, a, sigma, asa, g_r, t, info):
        self._count("newton_pspace")
        X = self._x_rows(op)
        idx = J[:p].numpy().astype(np.int64)
        Z = X[idx]
        aJ = a.numpy()[idx]
        P = np.eye(p) - (np.outer(aJ, aJ) / asa if asa != 0.0 else 0.0)
        M = np.eye(p) + sigma * P @ (Z @ Z.T) @ P
        y = np.linalg.solve(M, P @ grad.numpy()[idx])
        t.copy_(torch.from_numpy(-g_r.numpy() + sigma * Z.T @ (P @ y)))
        info[0] = 0

    def chol_solve(self, M, m, b, scale, x, info):
        self._count("chol_solve")
        Mh = M.numpy()
        try:
            L = np.linalg.cholesky(Mh)
        except np.linalg.LinAlgError:
            info[0] = 1
            return
        y = np.linalg.solve(L, scale * b.numpy())
        x.copy_(torch.from_numpy(np.linalg.solve(L.T, y)))
        info[0] = 0

    # sharded path --------------------------------------------------------------
    def proj_local(self, A, box, T, lam, mode, rec, B=None, coefs=None, x_out=None,
                   free_out=None, ref=None, base=None, base_lam=0.0):
        self._count("proj_local")
        a = box.a_dev.numpy()
        l = box.l.numpy()
        u = box.u.numpy()
        r = rec.view(-1, 8)
        for t in range(T):
            v = A.numpy().copy()
            if B is not None:
                v = v - float(coefs[t]) * B.numpy()
            y = v - lam[t] * a
            x = np.clip(y, l, u)
            if mode == 0:
                with np.errstate(divide="ignore", invalid="ignore"):
                    t1, t2 = (v - u) / a, (v - l) / a
                nz = a != 0
                b0, b1 = np.minimum(t1, t2)[nz], np.maximum(t1, t2)[nz]
                a2 = (a * a)[nz]
                right = np.where(b0 > lam[t], b0, np.where(b1 > lam[t], b1, np.inf))
                left = np.where(b1 < lam[t], b1, np.where(b0 < lam[t], b0, -np.inf))
                r[t, 0] = float(a @ x)
                r[t, 1] = float(a2[(b0 <= lam[t]) & (lam[t] < b1)].sum())
                r[t, 2] = float(a2[(b0 < lam[t]) & (lam[t] <= b1)].sum())
                r[t, 3] = float(right.min()) if right.size else np.inf
                r[t, 4] = float(left.max()) if left.size else -np.inf
            else:
                lower = y <= l + 1e-12 * (1.0 + np.abs(l))
                upper = ~lower & (y >= u - 1e-12 * (1.0 + np.abs(u)))
                free = ~(lower | upper)
                res = v - x
                r[t, 0] = (float(v @ v) if base is None
                           else _bregman(x, base, v, a, lam[t], base_lam))
                r[t, 1] = float(res @ res)
                r[t, 2] = float(((x - ref.numpy()) ** 2).sum()) if ref is not None else 0.0
                r[t, 3] = float((a[free] ** 2).sum())
                r[t, 4] = float(free.sum())
                r[t, 5] = float(x @ (2.0 * v - x))
                if x_out is not None:
                    x_out.view(-1, box.n)[t].copy_(torch.from_numpy(x))
                if free_out is not None:
                    free_out.view(-1, box.n)[t].copy_(torch.from_numpy(free.astype(np.uint8)))

    def sum_slices(self, k, src, out):
        self._count("sum_slices")
        sl = src.reshape(k, -1).numpy()
        acc = sl[0].copy()
        for j in range(1, k):
            acc = acc + sl[j]
        out.view(-1).copy_(torch.from_numpy(acc))

    def hs_apply_coef(self, free, a, y, beta, add, alpha, coef, out):
        self._count("hs_apply_coef")
        h = np.where(free.numpy().astype(bool), y.numpy() - coef * a.numpy(), 0.0)
        r = beta * h + (alpha * add.numpy() if add is not None else 0.0)
        out.copy_(torch.from_numpy(np.ascontiguousarray(r)))

    def qspace_assemble(self, m, u, asa, sigma, shift, M):
        self._count("qspace_assemble")
        G = M.numpy() - shift * np.eye(m)
        if u is not None and asa != 0.0:
            uu = u.numpy()
            G = G - np.outer(uu, uu) / asa
        M.copy_(torch.from_numpy(np.eye(m) + sigma * G))
