import sys, math, collections; sys.path.insert(0, '.')
import __graft_entry__ as g; g.build()
import paper_1910_01312_b200 as P
from paper_1910_01312_b200 import datagen, solver
cfg = datagen.config1()
pb = P.build_csvc_dual(cfg["A"], cfg["y"], cfg["C"])
hist = collections.Counter()
orig = solver._Engine.line_search
def ls(self, *a, **k):
    r = orig(self, *a, **k)
    hist[round(-math.log2(r[0]))] += 1
    return r
solver._Engine.line_search = ls
r = P.alm_solve(pb, P.AlmOptions(tol_kkt=1e-6), P.SsnOptions(engine="python"))
print(r.outer_iters, r.total_inner_iters, sorted(hist.items()), pb.engine().counters)
