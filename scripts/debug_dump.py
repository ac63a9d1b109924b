"""Write GPU factor dumps + level stats of a few cases to gpurun_out/ for offline analysis."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1603_09133_b200 as ce  # noqa: E402

out = os.path.join(ROOT, "gpurun_out")
os.makedirs(out, exist_ok=True)
cases = [(1, (0, 0, 0)), (2, (64, 64, 0)), (4, (16, 16, 16))]
if len(sys.argv) > 1:
    cases = [tuple(json.loads(a)) for a in sys.argv[1:]]
for cfg, grid in cases:
    p = ce.Problem(cfg, *grid)
    a = ce.DeviceMatrix(p.matrix())
    t = time.time()
    f = ce.ce_factorize(a, p.plan, p.strategy())
    wall = time.time() - t
    tag = f"cfg{cfg}_{'x'.join(str(g) for g in grid)}"
    f.dump(os.path.join(out, tag + ".bin"))
    x = np.random.default_rng(0).standard_normal(p.n)
    np.save(os.path.join(out, tag + "_solve.npy"), f.solve(x))
    t = time.time()
    for _ in range(3):
        f.solve(x)
    ts = (time.time() - t) / 3
    info = dict(stats=f.stats, levels=f.level_stats(), wall=wall, solve_s=ts)
    json.dump(info, open(os.path.join(out, tag + ".json"), "w"), indent=1)
    print(tag, json.dumps(info["stats"]), flush=True)
    for lv in info["levels"]:
        print("  ", {k: lv[k] for k in ("block_count", "max_block", "max_far_cols", "max_close", "seconds", "sweep_seconds")})
    print("  solve", ts)
