"""Quick end-to-end check on the GPU: cfg1 + shrunk cfg2 vs the oracle, with timings."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import paper_1603_09133_b200 as ce  # noqa: E402
from _dump import read_dump  # noqa: E402
from _oracle import OProblem  # noqa: E402
from _parity import compare, summarize  # noqa: E402

for cfg, grid in [(1, (0, 0, 0)), (2, (64, 64, 0)), (4, (16, 16, 16))]:
    t = time.time()
    p = ce.Problem(cfg, *grid)
    a = ce.DeviceMatrix(p.matrix())
    f = ce.ce_factorize(a, p.plan, p.strategy())
    print("cfg", cfg, grid, "gpu factor", f.stats, flush=True)
    op = OProblem.config(cfg, *grid)
    fo = op.factorize(eps=p.eps)
    f.dump("/tmp/g.bin")
    fo.dump("/tmp/o.bin")
    s = summarize(compare(read_dump("/tmp/g.bin"), read_dump("/tmp/o.bin")))
    print("parity", s, flush=True)
    x = np.random.default_rng(0).standard_normal(p.n)
    yg, yo = f.solve(x), fo.solve(x)
    print("solve rel", np.linalg.norm(yg - yo) / np.linalg.norm(yo), flush=True)
    rg, _ = ce.pcg(a, p.n, p.rhs, f, ce.PcgOptions(tol=p.tol))
    ro, _ = op.krylov(p.rhs, fo, tol=p.tol)
    print("pcg gpu", rg, "oracle", ro, "wall", time.time() - t, flush=True)
