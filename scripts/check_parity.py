"""Per-level GPU-vs-oracle parity summary for a few small cases (prints one line per level)."""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_1603_09133_b200 as ce  # noqa: E402
from _dump import read_dump  # noqa: E402
from _oracle import OProblem  # noqa: E402
from _parity import compare, summarize  # noqa: E402

cases = [(1, (0, 0, 0)), (2, (64, 64, 0)), (3, (64, 64, 0)), (4, (16, 16, 16))]
d = tempfile.mkdtemp()
for cfg, grid in cases:
    p = ce.Problem(cfg, *grid)
    op = OProblem.config(cfg, *grid)
    fo = op.factorize(eps=p.eps)
    fo.dump(os.path.join(d, "o.bin"))
    o = read_dump(os.path.join(d, "o.bin"))
    forced = [L["retained"].tolist() for L in o["levels"]]
    a = ce.DeviceMatrix(p.matrix())
    for mode in ("free", "forced"):
        f = ce.ce_factorize(a, p.plan, p.strategy(),
                            ce.FactorOptions(forced_ranks=forced if mode == "forced" else []))
        f.dump(os.path.join(d, "g.bin"))
        g = read_dump(os.path.join(d, "g.bin"))
        x = np.random.default_rng(0).standard_normal(p.n)
        ys, yo = f.solve(x), fo.solve(x)
        print(f"cfg{cfg} {grid} {mode}: levels g/o {len(g['levels'])}/{len(o['levels'])} tail {g['tail_dim']}/"
              f"{o['tail_dim']} solve_rel {np.linalg.norm(ys - yo) / np.linalg.norm(yo):.2e}", flush=True)
        for lv in range(min(len(g["levels"]), len(o["levels"]))):
            gg, oo = dict(g), dict(o)
            gg["levels"], oo["levels"] = g["levels"][lv:lv + 1], o["levels"][lv:lv + 1]
            gg["tail_dim"] = oo["tail_dim"] = 0
            s = summarize(compare(gg, oo))
            print(f"   L{lv} struct {s['structure_ok']} {s['mismatch'] or ''} sig {s['sigma_max']:.1e} "
                  f"rowmax {s['row_err_max']:.1e} p99 {s['row_err_p99']:.1e} le1e-10 {s['frac_le_1e10']:.3f} "
                  f"ill {s['illcond_rows']} {s['illcond_err_max']:.1e}", flush=True)
            if not s["structure_ok"]:
                break
