"""CSV reports of the reference CLI (proj/src/csv.cpp; cli.cpp:60-80,153-247) through the product
library's text builders (ce_fmt_double, ce_*_csv), the Python mirror (ce.CsvTable, ce.*_table) and
the C++ shim (include/ce_gpu.hpp).  Pins: tests/golden/csv_cfg1_64/ was written by the REFERENCE's own
cli.cpp / csv.cpp (scripts/make_csv_fixture.py, oracle/_ref); where oracle/_ref is built the live
reference functions are compared too.  The factor-backed tables are the -m gpu test at the end."""

import ctypes as C
import json
import os
import struct
import subprocess

import numpy as np
import pytest

import paper_1603_09133_b200 as ce
import _ref

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLD = os.path.join(HERE, "golden", "csv_cfg1_64")
VEC = json.load(open(os.path.join(GOLD, "format_vectors.json")))


def test_fmt_double_matches_reference_vectors():
    """fmt_double (csv.cpp:84-88): the shortest round-tripping text, as std::to_chars chooses it."""
    for hx, text in VEC["fmt_double"]:
        v = struct.unpack(">d", bytes.fromhex(hx))[0]
        assert ce.fmt_double(v) == text
        if np.isfinite(v):
            assert float(ce.fmt_double(v)) == v
    assert ce.fmt_index(-7) == "-7" and ce.fmt_index(2**40) == "1099511627776"


def test_describe_matches_reference_vectors():
    for (use_rank, rank, eps, absolute), text in VEC["describe"]:
        s = ce.CompressionStrategy.fixed_rank(rank) if use_rank else ce.CompressionStrategy.adaptive(eps, bool(absolute))
        assert s.describe() == text


@pytest.mark.skipif(not _ref.available(), reason="oracle/_ref not built")
def test_fmt_double_against_live_reference():
    L = _ref.lib()
    L.ceref_fmt_double.restype, L.ceref_fmt_double.argtypes = C.c_int, [C.c_double, C.c_char_p, C.c_int]
    buf = C.create_string_buffer(128)
    rng = np.random.default_rng(3)
    vals = np.concatenate([rng.standard_normal(500), np.exp(rng.uniform(-300, 300, 500)), rng.integers(0, 2**53, 200) * 1.0,
                           rng.integers(0, 10**6, 200) / 64.0])
    for v in vals:
        L.ceref_fmt_double(float(v), buf, 128)
        assert ce.fmt_double(float(v)) == buf.value.decode()


def test_csv_table_round_trip():
    """csv.hpp:11-13: parse followed by to_string reproduces the input bytes; empty cells and a
    missing final newline survive; empty text has no header row."""
    for name in ("factor_stats.csv", "factor_summary.csv", "solve_report.csv", "trace.csv"):
        text = open(os.path.join(GOLD, name)).read()
        t = ce.CsvTable.parse(text)
        assert t.to_string() == text
        assert all(len(r) == len(t.header) for r in t.rows)
    t = ce.CsvTable.parse("a,b,c\n1,,3\n,,\n")
    assert t.header == ["a", "b", "c"] and t.rows == [["1", "", "3"], ["", "", ""]]
    assert ce.CsvTable.parse("a,b\n1,2").to_string() == "a,b\n1,2\n"
    with pytest.raises(ValueError, match="no header row"):
        ce.CsvTable.parse("")


@pytest.mark.skipif(not _ref.available(), reason="oracle/_ref not built")
def test_csv_round_trip_against_live_reference():
    L = _ref.lib()
    L.ceref_csv_roundtrip.restype, L.ceref_csv_roundtrip.argtypes = C.c_int64, [C.c_char_p, C.c_char_p, C.c_int64]
    buf = C.create_string_buffer(4096)
    for text in ["a,b,c\n1,,3\n,,\n", "a,b\n1,2", "x\n", "h1,h2\n\n3,4\n", "a,,\n,,b\n"]:
        k = L.ceref_csv_roundtrip(text.encode(), buf, 4096)
        assert k >= 0 and ce.CsvTable.parse(text).to_string() == buf.value.decode()
    assert L.ceref_csv_roundtrip(b"", buf, 4096) < 0


def test_csv_table_files(tmp_path):
    t = ce.CsvTable(["n", "x"], [["1", ce.fmt_double(0.25)], ["2", ce.fmt_double(1e-9)]])
    p = str(tmp_path / "t.csv")
    t.write(p)
    assert open(p, "rb").read() == b"n,x\n1,0.25\n2,1e-09\n"
    assert ce.CsvTable.load(p) == t
    with pytest.raises(OSError, match="cannot open"):
        ce.CsvTable.load(str(tmp_path / "missing.csv"))


def test_solve_report_and_trace_tables_have_the_reference_layout():
    """Headers and cell formats of solve_report.csv / trace.csv equal the golden files' (cli.cpp:73-80,233-247);
    values written by the reference and re-formatted here reproduce its cells byte for byte."""
    gold = ce.CsvTable.load(os.path.join(GOLD, "trace.csv"))
    rep = ce.SolveReport(True, 2, 0.0, 0.0, 0.0,
                         [(int(r[0]), float(r[1]), float(r[2]), float(r[3])) for r in gold.rows])
    assert ce.trace_table(rep).to_string() == gold.to_string()
    gold = ce.CsvTable.load(os.path.join(GOLD, "solve_report.csv"))
    g = dict(zip(gold.header, gold.rows[0]))
    rep = ce.SolveReport(g["converged"] == "1", int(g["iterations"]), float(g["recurrence_resid"]),
                         float(g["true_resid"]), 0.0)
    t = ce.solve_report_table(int(g["n"]), g["mode"], ce.CompressionStrategy.adaptive(1e-4), True, rep,
                              float(g["factor_seconds"]), float(g["solve_seconds"]))
    assert t.to_string() == gold.to_string()
    none = ce.solve_report_table(16, "minres", None, False, rep, 0.0, 0.0)
    assert none.rows[0][2] == "none" and none.rows[0][3] == "0"


def test_shim_csv_program(tmp_path):
    """The C++ shim's CsvTable / fmt_double / describe / report tables (no GPU)."""
    exe = str(tmp_path / "shim_csv")
    lib = os.path.join(ROOT, "paper_1603_09133_b200")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), os.path.join(HERE, "shim_csv.cpp"),
                    "-o", exe, "-L", lib, "-lce_gpu", f"-Wl,-rpath,{lib}"], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.splitlines()
    assert out[0] == "0.1|1e+05|1e+22|-42"  # to_chars: the shorter of fixed and scientific
    assert out[1] == "eps=1e-06|abseps=0.0001|rank=8"
    assert out[2] == "iter,recurrence_resid,true_resid,seconds" and out[3] == "0,1,-1,0.001"
    assert out[5] == "2,1.5e-12,2.5e-12,0.003"
    assert out[7] == "4096,minres,eps=0.0001,1,1,2,1.5e-12,2.5e-12,0.25,0.5"
    assert out[9] == "4096,minres,none,0,1,2,1.5e-12,2.5e-12,0,0.5"
    assert out[10] == "csv text has no header row"
    for name in ("factor_stats.csv", "trace.csv"):
        src = os.path.join(GOLD, name)
        dst = str(tmp_path / name)
        open(dst, "wb").write(open(src, "rb").read())
        subprocess.run([exe, "roundtrip", dst], check=True, capture_output=True)
        assert open(dst + ".out", "rb").read() == open(src, "rb").read()


@pytest.mark.gpu
def test_factor_and_solve_reports_match_the_reference_cli(gpu_ctx, tmp_path):
    """run_factor / run_solve of the reference CLI (cli.cpp:153-247) on cfg1 at 64 x 64 as a `file`
    problem, against the GPU factorization of the same files: every structural cell (levels, eliminated
    unknowns, factor blocks, ranks, byte counts, predicted blocks, scalar nnz, iterations) identical;
    mean ranks and residual sizes agree; only the timings differ."""
    case = json.load(open(os.path.join(GOLD, "case.json")))
    p0 = ce.Problem(case["cfg"], *case["grid"])
    m, pl, r = (str(tmp_path / s) for s in ("matrix.mtx", "plan.txt", "rhs.txt"))
    p0.save(m, pl, r)
    p = ce.Problem.load(m, pl, r, block=case["block"])  # load_problem (cli.cpp:114-133)
    a = ce.DeviceMatrix(p.matrix())
    strat = ce.CompressionStrategy.adaptive(case["eps"])
    f = ce.ce_factorize(a, p.plan, strat, ce.FactorOptions(dense_threshold=case["dense_threshold"]))
    stats = ce.factor_stats_table(f)
    gold = ce.CsvTable.load(os.path.join(GOLD, "factor_stats.csv"))
    assert stats.header == gold.header and len(stats.rows) == len(gold.rows)
    for mine, ref in zip(stats.rows, gold.rows):
        for k, name in enumerate(gold.header):
            if name == "seconds":
                assert float(mine[k]) >= 0
            elif name == "mean_rank":
                assert mine[k] == ref[k]  # same ranks -> same mean, same shortest text
            else:
                assert mine[k] == ref[k], (name, mine, ref)
    summ = ce.factor_summary_table(f, case["block"], strat, f.stats["total_seconds"])
    gold = ce.CsvTable.load(os.path.join(GOLD, "factor_summary.csv"))
    assert summ.header == gold.header
    for k, name in enumerate(gold.header):
        if name in ("seconds", "recon_error"):
            continue
        assert summ.rows[0][k] == gold.rows[0][k], (name, summ.rows[0], gold.rows[0])
    rep, x = ce.minres(a, p.n, p.rhs, f, ce.MinresOptions(tol=case["tol"], maxit=case["maxit"]))
    tr = ce.trace_table(rep)
    gold = ce.CsvTable.load(os.path.join(GOLD, "trace.csv"))
    assert tr.header == gold.header and len(tr.rows) == len(gold.rows)
    assert tr.rows[0][:3] == gold.rows[0][:3]  # the iteration-0 sample: 0,1,1
    for mine, ref in zip(tr.rows[1:], gold.rows[1:]):
        assert mine[0] == ref[0]
        for k in (1, 2):  # residual histories agree to their leading digits (same operator, same factor)
            assert abs(float(mine[k]) - float(ref[k])) <= 0.05 * float(ref[k]) + 1e-13
    sr = ce.solve_report_table(p.n, "minres", strat, True, rep, f.stats["total_seconds"], rep.seconds)
    gold = ce.CsvTable.load(os.path.join(GOLD, "solve_report.csv"))
    assert sr.header == gold.header and sr.rows[0][:6] == gold.rows[0][:6]
