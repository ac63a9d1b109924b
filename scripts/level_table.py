"""Per-level sweep table (LevelStats + SURVEY §8d algorithmic counts + CUDA-event sweep time):
python scripts/level_table.py CFG PLAN [NX NY NZ] -> JSON lines, one per level, then a summary line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_09133_b200 as ce  # noqa: E402

cfg, plan = int(sys.argv[1]), sys.argv[2]
grid = [int(v) for v in sys.argv[3:6]] if len(sys.argv) >= 6 else []  # optional nx ny nz override
p = ce.Problem(cfg, *grid, plan=plan)
a = ce.DeviceMatrix(p.matrix())
for _ in range(2):
    f = ce.ce_factorize(a, p.plan, p.strategy())
st = f.stats
for lv, L in enumerate(f.level_stats()):
    t = L["sweep_seconds"]
    print(json.dumps({"level": lv + 1, "M": L["block_count"], "waves": L["n_waves"], "max_block": L["max_block"],
                      "max_close": L["max_close"], "sweep_ms": 1e3 * t, "level_ms": 1e3 * L["seconds"],
                      "alg_GB": L["algorithmic_bytes"] / 1e9, "GBs": L["algorithmic_bytes"] / t / 1e9 if t else 0,
                      "alg_TF": L["algorithmic_flops"] / 1e12, "TFs": L["algorithmic_flops"] / t / 1e12 if t else 0}))
print(json.dumps({"cfg": cfg, "plan": plan, "factor_s": st["device_seconds"], "sweep_s": st["sweep_kernel_seconds"],
                  "host_total_s": st["total_seconds"], "alg_GB": st["algorithmic_bytes"] / 1e9,
                  "alg_TF": st["algorithmic_flops"] / 1e12}))
