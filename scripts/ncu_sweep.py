"""One factorization of cfg2 at 256x256 (same stencil/B/eps) for an ncu --set full capture of the sweep kernel."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1603_09133_b200 as ce
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
p = ce.Problem(2, n, n, plan=os.environ.get("CE_PLAN", "reference"))
a = ce.DeviceMatrix(p.matrix())
f = ce.ce_factorize(a, p.plan, p.strategy())
print(f.stats)
