"""Dev aid: run the CUDA engine and the CPU test engine in lockstep on one golden SVM case."""
import sys; sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np, torch
import paper_1910_01312_b200 as P
from paper_1910_01312_b200 import svm, solver
from cpu_backend import CpuTestBackend
from conftest import load_cases
c = load_cases("solve.npz", "s")[int(sys.argv[1]) if len(sys.argv) > 1 else 11]
cpu = CpuTestBackend()
pg = svm.build_csvc_dual(c["A"], c["y"], c["C"])
pc = svm.build_csvc_dual(c["A"], c["y"], c["C"], backend=cpu)
eg, ec = pg.engine(), pc.engine()
rng = np.random.default_rng(0)
n = pg.n
for trial in range(3):
    x = rng.random(n) * c["C"] * (rng.random(n) < 0.3)
    w = rng.standard_normal(n) * 1e-2
    qw = pc.q_op.matvec(torch.from_numpy(w)).numpy()
    sigma = [1.0, 5.0, 125.0][trial]
    scg, curg = eg.start_inner(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), torch.from_numpy(qw).cuda(), sigma)
    scc, curc = ec.start_inner(torch.from_numpy(x), torch.from_numpy(w), torch.from_numpy(qw), sigma)
    print('start: sc', scg[:2], scc[:2], 'nfree', curg['nfree'], curc['nfree'], 'lam', curg['lam'], curc['lam'], 'asa', curg['sum_a2_free'], curc['sum_a2_free'])
    for name in ['u', 'xp', 's', 'grad']:
        a, b = getattr(eg, name).cpu().numpy(), getattr(ec, name).numpy()
        print('  ', name, np.abs(a - b).max(), np.abs(b).max())
    print('  free diff', (eg.free.cpu().numpy() != ec.free.numpy()).sum(), 'gr', np.abs(eg.gr[0].cpu().numpy() - ec.gr[0].numpy()).max())
    p = int(curg['nfree'])
    asa = float(curg['sum_a2_free']); eg.direction(p, sigma, asa); ec.direction(p, sigma, asa)
    sg, _ = eg.fetch(info=True); sc_, _ = ec.fetch(info=True)
    print('  dir dots', sg[:4], sc_[:4], 'info', int(eg.h_info[0]))
    for name in ['M', 'm1', 't', 'qdir', 'dir']:
        a, b = getattr(eg, name).cpu().numpy(), getattr(ec, name).numpy()
        if name == 'M':
            print('  ', name, 'diag/L?', a[:3, :3], b[:3, :3])
        print('  ', name, np.abs(a - b).max(), np.abs(b).max())
