import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_1603_09133_b200 as ce
from _dump import read_dump
from _oracle import OProblem
import json; cfg, nx = int(os.environ.get("FC_CFG", "1")), int(os.environ.get("FC_N", "32")); p = ce.Problem(cfg, nx, nx); a = ce.DeviceMatrix(p.matrix())
f = ce.ce_factorize(a, p.plan, p.strategy(), ce.FactorOptions(dense_threshold=64))
f.dump('/tmp/g.bin'); g = read_dump('/tmp/g.bin')
fo = OProblem.config(cfg, nx, nx).factorize(eps=p.eps, dense_threshold=64); fo.dump('/tmp/o.bin'); o = read_dump('/tmp/o.bin')
L, M = g['levels'][0], o['levels'][0]
print('mask', os.environ.get('CE_FORCE_TASKS'), 'levels', len(g['levels']), len(o['levels']), 'ranks g', L['retained'][:8], 'o', M['retained'][:8])
for b in range(1, 4): print('  row', b, 'sig g', np.round(L['sigma'][b], 6), 'o', np.round(M['sigma'][b], 6))
x = np.random.default_rng(0).standard_normal(p.n); print('  solve rel', np.linalg.norm(f.solve(x) - fo.solve(x)) / np.linalg.norm(fo.solve(x)))
print('  fcols g', L['fcols'][:6], 'o', M['fcols'][:6], 'has_basis g', L['has_basis'][:6], 'o', M['has_basis'][:6])
st = f.level_stats()[0]; print('  items', st['n_items'], 'waves', st['n_waves'])
