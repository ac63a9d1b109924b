"""Factorize the same problem several times and report the first (level, row, field)
where two runs differ bit-wise (race detector for the sweep kernel)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_1603_09133_b200 as ce  # noqa: E402
from _dump import read_dump  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nx = int(sys.argv[2]) if len(sys.argv) > 2 else 256
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
p = ce.Problem(cfg, nx, nx)
a = ce.DeviceMatrix(p.matrix())
dumps = []
for k in range(reps):
    f = ce.ce_factorize(a, p.plan, p.strategy())
    path = f"/tmp/det_{k}.bin"
    f.dump(path)
    dumps.append(read_dump(path))
    print("rep", k, "nnz", f.stats["l_scalar_nnz"], flush=True)


def first_diff(d0, d1):
    for li, (L0, L1) in enumerate(zip(d0["levels"], d1["levels"])):
        if not np.array_equal(L0["retained"], L1["retained"]):
            i = int(np.nonzero(L0["retained"] != L1["retained"])[0][0])
            return f"level {li + 1} row {i}: rank {L0['retained'][i]} vs {L1['retained'][i]}"
        for i in range(L0["m"]):
            s0, s1 = L0["sigma"][i], L1["sigma"][i]
            if len(s0) != len(s1) or not np.array_equal(s0, s1):
                return f"level {li + 1} row {i}: sigma differs (max {np.max(np.abs(s0 - s1)) if len(s0) == len(s1) else 'len'})"
            if L0["basis"][i] is not None and not np.array_equal(L0["basis"][i], L1["basis"][i]):
                return f"level {li + 1} row {i}: basis differs"
            r0, r1 = L0["rows"][i], L1["rows"][i]
            if (r0 is None) != (r1 is None):
                return f"level {li + 1} row {i}: width presence differs"
            if r0 is None:
                continue
            if not np.array_equal(r0["chol"], r1["chol"]):
                return f"level {li + 1} row {i}: chol differs"
            if not np.array_equal(r0["coupling"], r1["coupling"]):
                return f"level {li + 1} row {i}: coupling differs"
            for (t0, g0), (t1, g1) in zip(r0["neighbors"], r1["neighbors"]):
                if t0 != t1 or not np.array_equal(g0, g1):
                    return f"level {li + 1} row {i}: g of neighbour {t0} differs (max {np.max(np.abs(g0 - g1))})"
    return "identical"


def first_nan(d):
    for li, L in enumerate(d["levels"]):
        for i in range(L["m"]):
            if np.any(~np.isfinite(L["sigma"][i])):
                return f"level {li + 1} row {i} sigma {L['sigma'][i]}"
            r = L["rows"][i]
            if r is not None and not (np.all(np.isfinite(r["chol"])) and np.all(np.isfinite(r["coupling"]))):
                return f"level {li + 1} row {i} chol/coupling"
    return "none"


print("first non-finite:", first_nan(dumps[0]))
for k in range(1, reps):
    print("run 0 vs", k, ":", first_diff(dumps[0], dumps[k]), flush=True)
