"""Symbolic planner pieces on the device: pattern_square / coarsen_pattern
(proj/src/pattern.cpp:64-118) on the GPU against the oracle's restatement, entry for entry; and
the factorization that uses them for its first-level plan is unchanged (parity tests)."""

import numpy as np
import pytest

import paper_1603_09133_b200 as ce
import _oracle as O

pytestmark = pytest.mark.gpu


def _csr(rows):
    ptr = np.zeros(len(rows) + 1, np.int64)
    for i, r in enumerate(rows):
        ptr[i + 1] = ptr[i] + len(r)
    return ptr, np.array([c for r in rows for c in r] or [0], np.int64)[:ptr[-1]]


def _random_pattern(m, p, rng):
    a = rng.random((m, m)) < p
    a = a | a.T | np.eye(m, dtype=bool)
    return [sorted(np.nonzero(a[i])[0].tolist()) for i in range(m)]


@pytest.mark.parametrize("m,p,seed", [(1, 1.0, 0), (7, 0.3, 1), (60, 0.05, 2), (300, 0.01, 3), (200, 0.3, 4)])
def test_square_matches_oracle(gpu_ctx, m, p, seed):
    rows = _random_pattern(m, p, np.random.default_rng(seed))
    ptr, cols = _csr(rows)
    gp, gc = ce.pattern_square(ptr, cols)
    expect = O.pattern_op(0, rows)
    ep, ec = _csr(expect)
    assert np.array_equal(gp, ep) and np.array_equal(gc, ec)


@pytest.mark.parametrize("m,p,ng,seed", [(60, 0.05, 20, 5), (300, 0.02, 40, 6), (100, 0.2, 100, 7)])
def test_coarsen_matches_oracle(gpu_ctx, m, p, ng, seed):
    rng = np.random.default_rng(seed)
    rows = _random_pattern(m, p, rng)
    assign = rng.integers(0, ng, m)
    assign[:ng] = np.arange(ng)  # every group non-empty
    rng.shuffle(assign)
    ptr, cols = _csr(rows)
    gp, gc = ce.pattern_coarsen(ptr, cols, assign, ng)
    expect = O.pattern_op(2, rows, ng, assign)
    ep, ec = _csr(expect)
    assert np.array_equal(gp, ep) and np.array_equal(gc, ec)


def test_coarsen_drops_dead_groups(gpu_ctx):
    rows = _random_pattern(50, 0.1, np.random.default_rng(8))
    assign = np.arange(50) // 5  # 10 groups
    dead = assign.copy()
    dead[assign == 3] = -1  # group 3 dies: its rows and columns vanish
    ptr, cols = _csr(rows)
    gp, gc = ce.pattern_coarsen(ptr, cols, dead, 10)
    full = O.pattern_op(2, rows, 10, assign)
    for g in range(10):
        got = gc[gp[g]:gp[g + 1]].tolist()
        assert got == ([] if g == 3 else [c for c in full[g] if c != 3])


@pytest.mark.parametrize("cfg,grid", [(2, (256, 256, 0)), (3, (256, 256, 0)), (4, (32, 32, 32))])
def test_baseline_patterns(gpu_ctx, cfg, grid):
    """The BASELINE configs' level-1 block patterns (the oracle's dense output buffer bounds the size)."""
    p = ce.Problem(cfg, *grid)
    rows = [p.col_idx[p.row_ptr[i]:p.row_ptr[i + 1]].tolist() for i in range(p.m)]
    gp, gc = ce.pattern_square(p.row_ptr, p.col_idx)
    ep, ec = _csr(O.pattern_op(0, rows))
    assert np.array_equal(gp, ep) and np.array_equal(gc, ec)
