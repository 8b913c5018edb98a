"""The CG route's two products on config-3 data (n = 4M x q = 1M Zipf, |J| = 700k random
rows): python scripts/prof_sparse_kernels.py [reps].  Run under ncu for per-kernel times:
the restricted entry points rebuild the J-restricted copies on every call, the launch list
separates build and product kernels."""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import __graft_entry__ as g

g.build()
import paper_1910_01312_b200 as P
from paper_1910_01312_b200 import _lib, datagen
from paper_1910_01312_b200.operators import CsrKernelOperator

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
cfg = datagen.config3(n=int(4_000_000 * scale), q=int(1_000_000 * scale))
op = CsrKernelOperator((cfg["indptr"], cfg["indices"], cfg["data"], cfg["shape"]), labels=cfg["y"])
n, q = cfg["shape"]
rng = np.random.default_rng(5)
keep = (rng.random(n) < 0.175).astype(np.uint8)
J = np.flatnonzero(keep).astype(np.int32)
p = J.size
be = P.default_backend()
dev = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)
ws = be.zeros(int(_lib.load().ssnal_csr_restricted_ws_bytes(op._cref)), torch.uint8)
keep_d, J_d = dev(keep, torch.uint8), dev(np.r_[J, 0], torch.int32)
w_d, d_d = dev(rng.standard_normal(p)), dev(rng.standard_normal(q))
out, z = be.empty(q), be.empty(p)
nnzJ = int((cfg["indptr"][J + 1] - cfg["indptr"][J]).sum())
print(f"n={n} q={q} p={p} nnz(X_J)={nnzJ}", flush=True)
for _ in range(reps):
    _lib.call("ssnal_csr_xt_restricted", op._cref, keep_d.data_ptr(), J_d.data_ptr(), p,
              w_d.data_ptr(), out.data_ptr(), ws.data_ptr(), be.stream())
    _lib.call("ssnal_csr_xd_restricted", op._cref, keep_d.data_ptr(), J_d.data_ptr(), p,
              d_d.data_ptr(), z.data_ptr(), ws.data_ptr(), be.stream())
torch.cuda.synchronize()
# full products for comparison
v = dev(rng.standard_normal(n))
for _ in range(reps):
    op.xt([v])
    op.x(d_d.view(1, -1))
torch.cuda.synchronize()
print("done", float(out.sum()), float(z.sum()))
