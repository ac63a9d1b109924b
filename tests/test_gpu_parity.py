"""GPU-vs-oracle parity of the CE hot path, through the C-ABI.

Runs on a B200 only (-m gpu).  Sizes are chosen so the CPU oracle finishes in
seconds; the full-size configs are checked through size-independent
properties in test_gpu_fullsize.py.
"""

import os
import tempfile

import numpy as np
import pytest

import paper_1603_09133_b200 as ce
from _dump import read_dump
from _oracle import OProblem
from _parity import compare, summarize

pytestmark = pytest.mark.gpu

# (cfg, grid override) pairs: cfg1 at full size, the others shrunk.
CASES = [(1, (0, 0, 0)), (2, (64, 64, 0)), (3, (64, 64, 0)), (4, (16, 16, 16)), (5, (16, 16, 16))]


def _factor_both(cfg, grid, dense_threshold=2048):
    p = ce.Problem(cfg, *grid)
    op = OProblem.config(cfg, *grid)
    a = ce.DeviceMatrix(p.matrix())
    f = ce.ce_factorize(a, p.plan, p.strategy(), ce.FactorOptions(dense_threshold=dense_threshold))
    fo = op.factorize(eps=p.eps, dense_threshold=dense_threshold)
    return p, op, a, f, fo


def _dumps(f, fo):
    with tempfile.TemporaryDirectory() as d:
        gp, opth = os.path.join(d, "g.bin"), os.path.join(d, "o.bin")
        f.dump(gp)
        fo.dump(opth)
        return read_dump(gp), read_dump(opth)


@pytest.mark.parametrize("cfg,grid", CASES)
def test_factor_parity(gpu_ctx, cfg, grid):
    p, op, a, f, fo = _factor_both(cfg, grid, dense_threshold=512 if cfg in (4, 5) else 2048)
    g, o = _dumps(f, fo)
    rep = compare(g, o)
    s = summarize(rep)
    print(cfg, grid, s)
    assert s["structure_ok"], s["mismatch"]
    assert s["sigma_max"] <= 1e-13
    # canonical-gauge factor blocks: north-star tolerance 1e-10 relative Frobenius per row
    assert s["frac_le_1e10"] >= 0.99, s
    assert s["row_err_max"] <= 1e-7, s
    assert s["tail_err"] <= 1e-10


@pytest.mark.parametrize("cfg,grid", CASES)
def test_solve_and_pcg_parity(gpu_ctx, cfg, grid):
    p, op, a, f, fo = _factor_both(cfg, grid, dense_threshold=512 if cfg in (4, 5) else 2048)
    rng = np.random.default_rng(cfg)
    for _ in range(3):
        x = rng.standard_normal(p.n)
        yg, yo = f.solve(x), fo.solve(x)
        assert np.linalg.norm(yg - yo) <= 1e-10 * np.linalg.norm(yo)
        mg, mo = f.apply_operator(x), fo.apply_operator(x)
        assert np.linalg.norm(mg - mo) <= 1e-10 * np.linalg.norm(mo)
    rg, xg = ce.pcg(a, p.n, p.rhs, f, ce.PcgOptions(tol=p.tol, maxit=500))
    ro, xo = op.krylov(p.rhs, fo, "pcg", tol=p.tol, maxit=500)
    assert rg.converged and ro["converged"]
    assert abs(rg.iterations - ro["iterations"]) <= 1
    assert rg.final_true_residual <= 10 * p.tol
    # apply_q round trip
    x = rng.standard_normal(p.n)
    assert np.linalg.norm(f.apply_q_transpose(f.apply_q(x)) - x) <= 1e-12 * np.linalg.norm(x)
    np.testing.assert_allclose(f.apply_q(x), fo.apply_q(x), rtol=0, atol=1e-10 * np.abs(x).max())


def test_problem_matvec_parity(gpu_ctx):
    p = ce.Problem(2, 64, 64)
    op = OProblem.config(2, 64, 64)
    a = ce.DeviceMatrix(p.matrix())
    x = np.random.default_rng(0).standard_normal(p.n)
    np.testing.assert_allclose(a.matvec(x), op.matvec(x), rtol=1e-14, atol=1e-14)


def test_level_stats_match_oracle(gpu_ctx):
    p, op, a, f, fo = _factor_both(1, (0, 0, 0))
    gs, os_ = f.level_stats(), fo.level_stats()
    assert len(gs) == len(os_)
    for x, y in zip(gs, os_):
        for k in ("block_count", "pattern_blocks", "factor_blocks", "eliminated", "retained", "max_rank", "l_bytes",
                  "q_bytes"):
            assert x[k] == y[k], (k, x[k], y[k])
    st, so = f.stats, fo.summary()
    for k in ("factor_blocks", "predicted_factor_blocks", "l_scalar_nnz", "l_payload_bytes", "q_payload_bytes",
              "tail_bytes"):
        assert st[k] == so[k], (k, st[k], so[k])


def test_breakdown_negated_diagonal(gpu_ctx):
    """a negated diagonal entry -> BreakdownError at level 1."""
    p = ce.Problem(1, 32, 32)
    m = p.matrix()
    vals = m.values.copy()
    # negate scalar diagonal entry 0 of block 0
    vals[m.val_ptr[0]] = -vals[m.val_ptr[0]]
    bad = ce.BlockSparseMatrix(m.offsets, m.row_ptr, m.col_idx, m.val_ptr, vals)
    with pytest.raises(ce.BreakdownError) as ei:
        ce.ce_factorize(bad, p.plan, p.strategy(), ce.FactorOptions(dense_threshold=64))
    assert ei.value.level == 1
    assert ei.value.block == 0
