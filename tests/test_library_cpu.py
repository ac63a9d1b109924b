"""CPU-side checks of the product library (no GPU): it loads, exports every
C-ABI symbol include/ce_gpu.h declares, fails loudly without a device, and its
host-side BASELINE generator matches the oracle bit for bit."""

import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1603_09133_b200 as ce
from paper_1603_09133_b200 import _lib
from _oracle import OProblem

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ce_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ce_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    handle = C.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(handle, s)]
    assert not missing, missing
    # and the Python binding declares signatures for all of them
    assert set(syms) <= set(_lib.SIGNATURES), set(syms) - set(_lib.SIGNATURES)


def test_library_is_sm100a_cubin():
    """The .so carries sm_100a SASS (no PTX-JIT fallback target)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(ce.device_count() > 0, reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(RuntimeError, match="sm_100a GPU"):
        ce.Context(0)


@pytest.mark.parametrize("cfg,grid", [(1, (0, 0, 0)), (2, (64, 64, 0)), (3, (64, 64, 0)), (4, (16, 16, 16)),
                                      (5, (16, 16, 16)), (3, (96, 80, 0)), (5, (12, 8, 20))])
def test_generator_matches_oracle_bitwise(cfg, grid):
    """SURVEY.md §8d conventions: stencil, harmonic faces, RNG, ordering, plan -- identical CSB."""
    p = ce.Problem(cfg, *grid)
    o = OProblem.config(cfg, *grid)
    off, rp, ci, vp, vals = o.csb()
    assert np.array_equal(off, p.offsets)
    assert np.array_equal(rp, p.row_ptr)
    assert np.array_equal(ci, p.col_idx)
    assert np.array_equal(vp, p.val_ptr)
    assert np.array_equal(vals, p.values)  # bit-exact
    assert np.array_equal(o.rhs(), p.rhs)
    assert np.array_equal(o.perm(), p.perm)
    assigns, join = o.plan_assigns()
    assert join == p.plan.join and len(assigns) == len(p.plan.assigns)
    for x, y in zip(assigns, p.plan.assigns):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("plan", ["merge_all_axes", "merge_all_colored"])
@pytest.mark.parametrize("cfg,grid", [(2, (64, 32, 0)), (4, (16, 16, 16)), (5, (12, 8, 20)), (4, (32, 16, 8))])
def test_merge_all_axes_plan_matches_oracle(cfg, grid, plan):
    """CE_PLAN_MERGE_ALL_AXES / _COLORED: CSB, rhs, permutation and plan levels identical to the
    oracle's; every plan level groups at most 2^d blocks, and each axis halves per level until
    exhausted.  Uncoloured, the level-1 ordering is the reference plan's."""
    p = ce.Problem(cfg, *grid, plan=plan)
    r = ce.Problem(cfg, *grid)
    o = OProblem.config(cfg, *grid, plan=plan)
    off, rp, ci, vp, vals = o.csb()
    assert np.array_equal(rp, p.row_ptr) and np.array_equal(ci, p.col_idx) and np.array_equal(vals, p.values)
    assert np.array_equal(o.rhs(), p.rhs) and np.array_equal(o.perm(), p.perm)
    if plan == "merge_all_axes":
        assert np.array_equal(p.values, r.values) and np.array_equal(p.perm, r.perm)
    assigns, join = o.plan_assigns()
    assert join == p.plan.join == 2 and len(assigns) == len(p.plan.assigns)
    for x, y in zip(assigns, p.plan.assigns):
        assert np.array_equal(x, y)
    d = 3 if cfg in (4, 5) else 2
    for a in p.plan.assigns:
        assert np.bincount(a).max() <= 2 ** d
    assert len(p.plan.assigns) < len(r.plan.assigns)
    if plan == "merge_all_colored":  # one colour's blocks share no squared-pattern entry (level 1)
        import scipy.sparse as sp
        rows = np.repeat(np.arange(p.m), np.diff(p.row_ptr))
        B = sp.csr_matrix((np.ones(len(rows)), (rows, p.col_idx)), shape=(p.m, p.m))
        S = (B @ B).tocoo()
        first = p.perm[p.offsets[:-1]]
        # colour of each block from the cell containing its first unknown
        sh = {2: (4, 4, 1), 4: (4, 4, 2), 5: (4, 4, 2)}[cfg]
        x, y = first % grid[0], (first // grid[0]) % grid[1]
        z = first // (grid[0] * grid[1]) if d == 3 else 0 * x
        col = (x // sh[0]) % 3 + 3 * ((y // sh[1]) % 3) + 9 * ((z // sh[2]) % 3)
        assert np.all(np.diff(col) >= 0)  # colour-major
        off_diag = S.row != S.col
        assert not np.any(col[S.row[off_diag]] == col[S.col[off_diag]])
    with pytest.raises(ValueError):
        ce.Problem(cfg, *grid, plan="nope")


def test_generator_sizes_match_baseline_configs():
    """BASELINE.json configs: n and block size."""
    expect = {1: (16384, 8), 2: (1048576, 16)}
    for cfg, (n, b) in expect.items():
        p = ce.Problem(cfg)
        assert p.n == n and p.block == b
        assert int(np.max(np.diff(p.offsets))) == b


def test_random_k_is_lognormal_and_symmetric():
    p = ce.Problem(3, 64, 64)
    a = p.matrix()
    # symmetric blocks: (i,j) == (j,i)^T exactly
    for i in range(0, a.m, 7):
        for k in range(a.row_ptr[i], a.row_ptr[i + 1]):
            j = a.col_idx[k]
            kk = a.row_ptr[j] + int(np.searchsorted(a.col_idx[a.row_ptr[j]:a.row_ptr[j + 1]], i))
            bi = np.diff(a.offsets)[i]
            bj = np.diff(a.offsets)[j]
            x = a.values[a.val_ptr[k]:a.val_ptr[k + 1]].reshape(bi, bj)
            y = a.values[a.val_ptr[kk]:a.val_ptr[kk + 1]].reshape(bj, bi)
            assert np.array_equal(x, y.T)
