"""bench.py's JSON-line contract: the reference arm runs on CPU (the oracle port), so its line is
checked here without a GPU; the product arm's line is checked on a B200 (-m gpu) on cfg1."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "config", "e2e"}


def _run(args, env=None):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=dict(os.environ, **(env or {})))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--cfg", "1", "--steps", "1", "--warmup", "1", "--ref-threads", "2"])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["cfg"] == 1
    assert "CPU sample actually timed" in d["config"]["workload"]


@pytest.mark.gpu
def test_product_line_cfg1():
    d = _run(["--cfg", "1", "--steps", "2", "--warmup", "3", "--e2e-steps", "1", "--no-cpu-baseline", "--no-extra"])
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["dtype"] == "f64"
    assert d["pcg_converged"] and d["pcg_iterations"] <= 3
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r) and 0 < r["frac"] < 1
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] == 8 * d["config"]["n"]
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    v = d["plan_variant"]
    assert v["plan"] == "merge_all_colored" and v["value"] > 0 and v["pcg_converged"]
    ra = d["roofline_apply"]
    assert ra["bound"] == "hbm" and ra["algorithmic_bytes"] > 0 and 0 < ra["frac"] < 1 and ra["matvec"]["ms"] > 0
    assert d["validate"]["max_orth_error"] <= 1e-12 and d["validate"]["seconds"] > 0
    assert "extra_configs" not in d
    sh = d["sharded"]
    assert "error" not in sh, sh
    assert sh["value"] > 0 and sh["scaling"] == "strong" and sh["interior_rows"] > 0


@pytest.mark.gpu
def test_product_line_two_ranks_one_gpu():
    """bench.py's N > 1 code path (barriers, max-over-ranks, the sharded factorization's
    exchanges) with 2 ranks on the test box's one GPU over gloo."""
    port = 29500 + os.getpid() % 1000
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--cfg", "1",
           "--steps", "2", "--warmup", "3", "--e2e-steps", "1", "--no-cpu-baseline", "--no-extra", "--no-variants"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT,
                         env=dict(os.environ, CE_BENCH_SAME_DEVICE="1", CE_BENCH_BACKEND="gloo"))
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    sh = d["sharded"]
    assert "error" not in sh, sh
    assert sh["n_gpus"] == 2 and sh["own_rows_rank0"] < sh["interior_rows"] and sh["exchange_bytes_rank0"] > 0
