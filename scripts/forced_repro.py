import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_1603_09133_b200 as ce
from _dump import read_dump
import _oracle as O
cfg = int(sys.argv[1]); n = int(sys.argv[2])
p = ce.Problem(cfg, n, n); op = O.OProblem.config(cfg, n, n)
fo = op.factorize(eps=p.eps); fo.dump('/tmp/o.bin'); o = read_dump('/tmp/o.bin')
forced = [L['retained'].tolist() for L in o['levels']]
a = ce.DeviceMatrix(p.matrix())
f = ce.ce_factorize(a, p.plan, p.strategy(), ce.FactorOptions(forced_ranks=forced))
print('ok', f.stats['n_levels'], f.stats['tail_dim'], len(o['levels']), o['tail_dim'])
g = ce.ce_factorize(a, p.plan, p.strategy())
print('free ok')
f2 = ce.ce_factorize(a, p.plan, p.strategy(), ce.FactorOptions(forced_ranks=forced))
print('forced after free ok')
