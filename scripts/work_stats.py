"""Per-level work of one cfg factorization (ranks / flops / bytes) to separate code speed
from changes in the (chaotic) factorization structure when A/B-testing variants."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1603_09133_b200 as ce
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
p = ce.Problem(cfg)
a = ce.DeviceMatrix(p.matrix())
f = ce.ce_factorize(a, p.plan, p.strategy())
st = f.stats
print("nnz", st["l_scalar_nnz"], "GFLOP", round(st["algorithmic_flops"] / 1e9, 1), "GB", round(st["algorithmic_bytes"] / 1e9, 1))
print(" ".join(f"{i+1}:{s['retained']}/{s['sweep_seconds']*1e3:.0f}ms" for i, s in enumerate(f.level_stats())))
