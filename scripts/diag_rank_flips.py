"""Per-level free-run rank differences GPU vs oracle, with sigma_k / threshold of the differing
rows, and the preconditioner-apply deviation (development tool; found the oracle's Householder
overflow on roundoff columns).  Edit cfg / grid / plan below."""
import sys, os, tempfile
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import paper_1603_09133_b200 as ce
import _oracle as O
from _dump import read_dump
cfg, grid, dth, plan = 1, (0, 0, 0), 256, "merge_all_colored"
p = ce.Problem(cfg, *grid, plan=plan)
op = O.OProblem.config(cfg, *grid, plan=plan)
fo = op.factorize(eps=p.eps, dense_threshold=dth)
d = tempfile.mkdtemp()
fo.dump(d + "/o.bin"); o = read_dump(d + "/o.bin")
a = ce.DeviceMatrix(p.matrix())
g = ce.ce_factorize(a, p.plan, p.strategy(), ce.FactorOptions(dense_threshold=dth))
g.dump(d + "/g.bin"); gd = read_dump(d + "/g.bin")
for lv, (L, G) in enumerate(zip(o["levels"], gd["levels"])):
    diff = np.nonzero(L["retained"] != G["retained"])[0]
    print("level", lv + 1, "rows", len(L["retained"]), "rank diffs", len(diff))
    for i in diff[:10]:
        s = L["sigma"][i]; sg = G["sigma"][i]
        thr = p.eps * s[0] if len(s) else 0
        r_o, r_g = L["retained"][i], G["retained"][i]
        k = min(r_o, r_g)
        print("  row", i, "ranks o/g", r_o, r_g, "sigma_k/thr o", s[k] / thr if k < len(s) else None,
              "g", sg[k] / (p.eps * sg[0]) if k < len(sg) else None, "s1", s[0])
x = np.random.default_rng(7).standard_normal(p.n)
print("solve rel diff", np.linalg.norm(g.solve(x) - fo.solve(x)) / np.linalg.norm(fo.solve(x)))
