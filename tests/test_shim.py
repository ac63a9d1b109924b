"""The header-only C++ shim (include/ce_gpu.hpp) compiles against the C-ABI and, on a GPU,
runs the reference call shapes (ce_factorize -> solve as PCG preconditioner)."""

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1603_09133_b200")


def _build(tmp_path, src="shim_smoke.cpp"):
    exe = str(tmp_path / src.replace(".cpp", ""))
    subprocess.run(["g++", "-std=c++17", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", src), os.path.join(LIBDIR, "libce_gpu.so"), f"-Wl,-rpath,{LIBDIR}",
                    "-o", exe], check=True)
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


def test_reference_binding_compiles_and_maps_no_gpu_to_exit_1(tmp_path):
    """INTEGRATION.md's binding: ce::Vector / ce::BreakdownError through the shim's customisation
    points, ApplyFn minres/pcg call shapes (cli.cpp:198,225-226); without a GPU guarded() returns 1."""
    import paper_1603_09133_b200 as ce
    exe = _build(tmp_path, "shim_reference_binding.cpp")
    if ce.device_count() == 0:
        r = subprocess.run([exe], capture_output=True, text=True)
        assert r.returncode == 1 and "sm_100a GPU" in r.stdout


@pytest.mark.gpu
def test_reference_binding_solves_on_gpu(tmp_path):
    exe = _build(tmp_path, "shim_reference_binding.cpp")
    r = subprocess.run([exe, "solve"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "binding ok" in r.stdout


@pytest.mark.gpu
def test_reference_binding_breakdown_is_exit_2(tmp_path):
    """A negated diagonal raises ce::BreakdownError through the shim, which the
    reference's guarded() (cli.cpp:82-95) maps to exit code 2."""
    exe = _build(tmp_path, "shim_reference_binding.cpp")
    r = subprocess.run([exe, "breakdown"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 2, r.stdout + r.stderr
    assert "level 1, block 0" in r.stdout
