"""One small factorization + apply (development tool for debug builds with device asserts):
python scripts/sanitize_small.py [cfg] [n] [plan]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1603_09133_b200 as ce  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32
plan = sys.argv[3] if len(sys.argv) > 3 else "reference"
p = ce.Problem(cfg, n, n, n if cfg >= 4 else 0, plan=plan)
a = ce.DeviceMatrix(p.matrix())
f = ce.ce_factorize(a, p.plan, p.strategy(), ce.FactorOptions(dense_threshold=128))
y = f.solve(np.ones(p.n))
print("ok", p.n, f.stats["n_levels"], float(np.linalg.norm(y)))
