"""The header-only C++ shim (include/ce_gpu.hpp) compiles against the C-ABI and, on a GPU,
runs the reference call shapes (ce_factorize -> solve as PCG preconditioner)."""

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1603_09133_b200")


def _build(tmp_path):
    exe = str(tmp_path / "shim_smoke")
    subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "shim_smoke.cpp"),
                    os.path.join(LIBDIR, "libce_gpu.so"), f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_shim_compiles_and_fails_loudly_without_gpu(tmp_path):
    import paper_1603_09133_b200 as ce
    exe = _build(tmp_path)
    if ce.device_count() == 0:
        r = subprocess.run([exe], capture_output=True, text=True)
        assert r.returncode == 2 and "sm_100a GPU" in r.stdout


@pytest.mark.gpu
def test_shim_runs_on_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "shim ok" in r.stdout
