import sys; sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np
import paper_1910_01312_b200 as P
from conftest import load_cases
for i, c in enumerate(load_cases("solve.npz", "s")):
    if c["kind"] == "dense":
        pb = P.QpProblem(P.DenseOperator(c["G"].T @ c["G"]), c["c"], P.BoxLineSet(c["a"], c["d"], c["l"], c["u"]))
    elif c["kind"] == "csvc":
        pb = P.build_csvc_dual(c["A"], c["y"], c["C"])
    else:
        pb = P.build_svr_dual(c["A"], c["t"], c["C"], c["eps"])
    r = P.alm_solve(pb, P.AlmOptions(tol_kkt=c["tol"]))
    print(i, c["kind"], r.converged, c["converged"], "%.3e %.3e" % (r.kkt_residual, c["kkt"]), r.outer_iters, c["outer"], r.total_inner_iters, c["inner"], "%.2e" % (r.objective - c["obj"]), "%.2e" % np.abs(r.x_opt - c["x_opt"]).max(), "%.3fs" % r.wall_time, r.warnings[-1:] )
