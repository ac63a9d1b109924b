"""Compare the factor of two library builds on one small case, level by level (development tool).
usage: python scripts/cmp_builds.py LIB_A LIB_B CFG NX NY [NZ]   (run under gpurun)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

code = """
import sys, json, numpy as np
sys.path.insert(0, %r)
import paper_1603_09133_b200 as ce
cfg = int(sys.argv[2]); grid = [int(v) for v in sys.argv[3:]]
p = ce.Problem(cfg, *grid)
a = ce.DeviceMatrix(p.matrix())
f = ce.ce_factorize(a, p.plan, p.strategy(), ce.FactorOptions(dense_threshold=64))
f.dump(sys.argv[1])
"""
libs = sys.argv[1:3]
args = sys.argv[3:]
paths = []
for k, lib in enumerate(libs):
    path = "/tmp/cmp_%d.bin" % k
    env = dict(os.environ)
    if lib != "default":
        env["CE_LIB_OVERRIDE"] = lib
    r = subprocess.run([sys.executable, "-c", code % ROOT, path] + args, env=env, capture_output=True, text=True)
    print(lib, "rc", r.returncode, r.stderr.strip().splitlines()[-1:] if r.returncode else "")
    paths.append(path if r.returncode == 0 else None)
if None in paths:
    sys.exit(0)
from _dump import read_dump  # noqa: E402

A, B = read_dump(paths[0]), read_dump(paths[1])
print("levels", len(A["levels"]), len(B["levels"]))
for l, (LA, LB) in enumerate(zip(A["levels"], B["levels"])):
    ra, rb = np.asarray(LA["retained"]), np.asarray(LB["retained"])
    same = ra.shape == rb.shape and np.array_equal(ra, rb)
    msg = "level %d: M %d ranks %s" % (l + 1, len(ra), "equal" if same else "DIFFER")
    if not same and ra.shape == rb.shape:
        bad = np.nonzero(ra != rb)[0]
        msg += " first rows %s a %s b %s" % (bad[:8].tolist(), ra[bad[:8]].tolist(), rb[bad[:8]].tolist())
    print(msg)
    if not same:
        break
    # row factor values (chol, coupling, neighbour slices) and bases
    worst, wrow, wkey = 0.0, -1, ""
    def upd(va, vb, i, key):
        global worst, wrow, wkey
        va, vb = np.asarray(va, dtype=float), np.asarray(vb, dtype=float)
        if va.shape != vb.shape:
            print("  row", i, key, "shape", va.shape, vb.shape)
            return
        if va.size:
            d = float(np.max(np.abs(va - vb)))
            if not np.isfinite(d):
                d = float("inf")
            if d > worst:
                worst, wrow, wkey = d, i, key
    for i, (qa, qb) in enumerate(zip(LA["rows"], LB["rows"])):
        if LA["basis"][i] is not None and LB["basis"][i] is not None:
            upd(LA["basis"][i], LB["basis"][i], i, "basis")
        if qa is None or qb is None:
            continue
        upd(qa["chol"], qb["chol"], i, "chol")
        upd(qa["coupling"], qb["coupling"], i, "coupling")
        for (ta, ga), (tb, gb) in zip(qa["neighbors"], qb["neighbors"]):
            upd(ga, gb, i, "g[%d]" % ta)
    print("  max |a - b| over bases / row factors %.3e at row %d (%s)" % (worst, wrow, wkey))
