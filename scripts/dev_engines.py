import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import __graft_entry__ as g; g.build()
import paper_1910_01312_b200 as P
from conftest import load_cases
for i, c in enumerate(load_cases("solve.npz", "s")):
    for psi in ("reference", "stable"):
        out = []
        for eng in ("native", "python"):
            if c["kind"] == "dense":
                pb = P.QpProblem(P.DenseOperator(c["G"].T @ c["G"]), c["c"], P.BoxLineSet(c["a"], c["d"], c["l"], c["u"]))
            elif c["kind"] == "csvc":
                pb = P.build_csvc_dual(c["A"], c["y"], c["C"])
            else:
                pb = P.build_svr_dual(c["A"], c["t"], c["C"], c["eps"])
            rows = []
            r = P.alm_solve(pb, P.AlmOptions(tol_kkt=c["tol"]), P.SsnOptions(psi_eval=psi, engine=eng), callback=lambda *a: rows.append(a))
            out.append((r.converged, r.outer_iters, r.total_inner_iters, r.kkt_residual, r.objective, len(rows)))
        print(i, c["kind"], psi, "golden", c["converged"], c["outer"], c["inner"], "|", out[0], "|", out[1], "SAME" if out[0] == out[1] else "DIFF")
