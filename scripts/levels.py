"""Factorize one config on the GPU and print per-level stats + timings (no dumps)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1603_09133_b200 as ce  # noqa: E402

cfg = int(sys.argv[1])
grid = [int(x) for x in sys.argv[2:5]] if len(sys.argv) > 4 else [0, 0, 0]
t = time.time()
p = ce.Problem(cfg, *grid, plan=os.environ.get("CE_PLAN", "reference"))
print("gen", time.time() - t, "n", p.n, flush=True)
a = ce.DeviceMatrix(p.matrix())
for rep in range(2):
    t = time.time()
    f = ce.ce_factorize(a, p.plan, p.strategy())
    print("factor wall", time.time() - t, json.dumps(f.stats), flush=True)
for lv in f.level_stats():
    print("  ", {k: (round(v, 5) if isinstance(v, float) else v) for k, v in lv.items()
                 if k in ("block_count", "max_block", "max_far_cols", "max_close", "eliminated", "retained", "seconds",
                          "sweep_seconds", "max_rank", "n_waves", "pattern_blocks", "n_items")}, flush=True)
t = time.time()
rep, x = ce.pcg(a, p.n, p.rhs, f, ce.PcgOptions(tol=p.tol))
print("pcg", rep, "wall", time.time() - t, flush=True)
xx = np.random.default_rng(0).standard_normal(p.n)
t = time.time()
for _ in range(3):
    f.solve(xx)
print("apply ms", (time.time() - t) / 3 * 1e3, flush=True)
