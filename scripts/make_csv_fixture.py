"""Golden CSV reports from the REFERENCE's own CLI code (oracle/_ref: cli.cpp / csv.cpp compiled
unmodified): run_factor + run_solve on the `file` problem the product generator saves for cfg1 at
64 x 64, plus fmt_double / describe vectors.  Run here (needs /root/reference to build oracle/_ref);
the outputs under tests/golden/ travel to the GPU box.  usage: python scripts/make_csv_fixture.py"""
import ctypes as C
import json
import os
import struct
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1603_09133_b200 as ce  # noqa: E402
import _ref  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "csv_cfg1_64")


def fmt_values():
    rng = np.random.default_rng(7)
    v = [0.0, -0.0, 1.0, -1.0, 0.1, 0.5, 1e-6, 1e-5, 1e-4, 1e-3, 100000.0, 1e15, 1e16, 1e21, 1e22, 123456.789,
         2.5e-10, 1.0 / 3.0, 15.342, 4096.0, 5e-324, 1.7976931348623157e308, float("inf"), float("-inf")]
    v += list(rng.standard_normal(40)) + list(np.exp(rng.uniform(-40, 40, 40))) + list(rng.integers(0, 10**9, 10) / 8.0)
    return [float(x) for x in v]


def main():
    L = _ref.lib()
    L.ceref_fmt_double.restype, L.ceref_fmt_double.argtypes = C.c_int, [C.c_double, C.c_char_p, C.c_int]
    L.ceref_describe.restype = C.c_int
    L.ceref_describe.argtypes = [C.c_int, C.c_int64, C.c_double, C.c_int, C.c_char_p, C.c_int]
    L.ceref_run_factor.restype = C.c_int
    L.ceref_run_factor.argtypes = [C.c_char_p] * 3 + [C.c_int64, C.c_int, C.c_int64, C.c_double, C.c_int, C.c_int64,
                                                      C.c_char_p]
    L.ceref_run_solve.restype = C.c_int
    L.ceref_run_solve.argtypes = [C.c_char_p] * 3 + [C.c_int64, C.c_int, C.c_int64, C.c_double, C.c_int, C.c_int64,
                                                     C.c_double, C.c_int64, C.c_int, C.c_int, C.c_char_p]
    buf = C.create_string_buffer(256)
    vec = []
    for v in fmt_values():
        L.ceref_fmt_double(v, buf, 256)
        vec.append([struct.pack(">d", v).hex(), buf.value.decode()])
    desc = []
    for args in [(0, 0, 1e-6, 0), (0, 0, 1e-4, 1), (1, 8, 0.0, 0), (0, 0, 0.00012345678, 0), (0, 0, 2.5, 0)]:
        L.ceref_describe(*args, buf, 256)
        desc.append([list(args), buf.value.decode()])
    os.makedirs(OUT, exist_ok=True)
    json.dump({"fmt_double": vec, "describe": desc}, open(os.path.join(OUT, "format_vectors.json"), "w"), indent=0)

    p = ce.Problem(1, 64, 64)
    with tempfile.TemporaryDirectory() as d:
        m, pl, r = (os.path.join(d, s).encode() for s in ("matrix.mtx", "plan.txt", "rhs.txt"))
        p.save(m.decode(), pl.decode(), r.decode())
        rc = L.ceref_run_factor(m, r, pl, p.block, 0, 0, p.eps, 0, 256, OUT.encode())
        assert rc == 0, rc
        rc = L.ceref_run_solve(m, r, pl, p.block, 0, 0, p.eps, 0, 256, p.tol, 200, 0, 0, OUT.encode())
        assert rc == 0, rc
    os.remove(os.path.join(OUT, "x.txt"))
    json.dump({"cfg": 1, "grid": [64, 64, 0], "dense_threshold": 256, "block": int(p.block), "eps": p.eps,
               "tol": p.tol, "maxit": 200}, open(os.path.join(OUT, "case.json"), "w"))
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
