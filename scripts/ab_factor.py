"""Factor-time A/B of library builds (CE_LIB_OVERRIDE), CUDA events on the library stream.
usage: python scripts/ab_factor.py CFG PLAN STEPS   (library chosen by CE_LIB_OVERRIDE)"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1603_09133_b200 as ce  # noqa: E402
from paper_1603_09133_b200._lib import lib  # noqa: E402

cfg, plan, steps = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
p = ce.Problem(cfg, plan=plan)
ctx = ce.Context.get(0)
a = ce.DeviceMatrix(p.matrix(), ctx)
sp = C.c_void_p()
lib.ce_ctx_stream(ctx.handle, C.byref(sp))
stream = torch.cuda.ExternalStream(sp.value, device="cuda:0")
b = torch.from_numpy(p.rhs).cuda()
out = []
for k in range(steps + 1):
    with torch.cuda.stream(stream):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        f = ce.ce_factorize(a, p.plan, p.strategy(), ce.FactorOptions(), ctx)
        e1.record(stream)
        rep, x = ce.pcg(a, p.n, b, f, ce.PcgOptions(tol=p.tol))
        e2.record(stream)
    e2.synchronize()
    if k:
        out.append((round(e0.elapsed_time(e1), 1), round(e1.elapsed_time(e2), 1), rep.iterations))
    del f
print(json.dumps({"lib": os.environ.get("CE_LIB_OVERRIDE", "default"), "cfg": cfg, "plan": plan, "steps": out}))
