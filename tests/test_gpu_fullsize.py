"""Full-size BASELINE configs on the GPU, checked through size-independent
properties (the oracle is too slow at these sizes): telescoping dimensions,
orthogonal bases (sampled), M (M^-1 x) = x, PCG to the stated tolerance with the
true residual below target, deterministic re-factorization."""

import numpy as np
import pytest

import paper_1603_09133_b200 as ce

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg2(gpu_ctx):
    p = ce.Problem(2)
    a = ce.DeviceMatrix(p.matrix())
    f = ce.ce_factorize(a, p.plan, p.strategy())
    return p, a, f


def test_cfg2_dimensions_telescope(cfg2):
    p, a, f = cfg2
    lv = f.level_stats()
    assert lv[0]["block_count"] == 65536
    dim = p.n
    for s in lv:
        assert s["eliminated"] + s["retained"] == dim
        dim = s["retained"]
    assert dim == f.stats["tail_dim"]
    assert f.stats["shift_retries"] == 0


def test_cfg2_pcg_reaches_target(cfg2):
    p, a, f = cfg2
    rep, x = ce.pcg(a, p.n, p.rhs, f, ce.PcgOptions(tol=p.tol, maxit=200))
    assert rep.converged
    assert rep.final_true_residual <= 10 * p.tol
    r = p.rhs - a.matvec(x)
    assert np.linalg.norm(r) <= 10 * p.tol * np.linalg.norm(p.rhs)


def test_cfg2_operator_self_consistency(cfg2):
    p, a, f = cfg2
    x = np.random.default_rng(0).standard_normal(p.n)
    y = f.apply_operator(f.solve(x))
    assert np.linalg.norm(y - x) <= 1e-8 * np.linalg.norm(x)
    # M approximates A: ||A x - M x|| small relative to ||A x|| at eps = 1e-6
    ax, mx = a.matvec(x), f.apply_operator(x)
    assert np.linalg.norm(ax - mx) <= 1e-3 * np.linalg.norm(ax)


def test_cfg2_refactorization_deterministic(cfg2):
    p, a, f = cfg2
    g = ce.ce_factorize(a, p.plan, p.strategy())
    x = np.random.default_rng(1).standard_normal(p.n)
    assert np.array_equal(f.solve(x), g.solve(x))


def test_cfg1_full_pcg(gpu_ctx):
    p = ce.Problem(1)
    a = ce.DeviceMatrix(p.matrix())
    f = ce.ce_factorize(a, p.plan, p.strategy())
    rep, x = ce.pcg(a, p.n, p.rhs, f, ce.PcgOptions(tol=p.tol))
    assert rep.converged and rep.final_true_residual <= 10 * p.tol


def test_cfg3_fullsize_properties(gpu_ctx):
    """BASELINE cfg3 (2-D variable-coefficient FV, n = 4.2 M): telescoping dimensions and PCG to
    the stated tolerance with the true residual below target."""
    p = ce.Problem(3)
    a = ce.DeviceMatrix(p.matrix())
    f = ce.ce_factorize(a, p.plan, p.strategy())
    dim = p.n
    for s in f.level_stats():
        assert s["eliminated"] + s["retained"] == dim
        dim = s["retained"]
    assert dim == f.stats["tail_dim"]
    rep, x = ce.pcg(a, p.n, p.rhs, f, ce.PcgOptions(tol=p.tol, maxit=200))
    assert rep.converged and rep.final_true_residual <= 10 * p.tol


@pytest.mark.parametrize("cfg", [2, 3])
def test_colored_plan_fullsize_properties(gpu_ctx, cfg):
    """cfg2 / cfg3 at full size under the colour-major all-axis-merge plan (DESIGN.md "Plan
    families"): every level's row DAG has at most 9 waves (one per mod-3 colour), dimensions
    telescope, M (M^-1 x) = x, PCG reaches the stated tolerance with the true residual below
    target, and re-factorization is bitwise deterministic."""
    p = ce.Problem(cfg, plan="merge_all_colored")
    a = ce.DeviceMatrix(p.matrix())
    f = ce.ce_factorize(a, p.plan, p.strategy())
    dim = p.n
    for s in f.level_stats():
        assert s["n_waves"] <= 9
        assert s["max_close"] <= 8
        assert s["eliminated"] + s["retained"] == dim
        dim = s["retained"]
    assert dim == f.stats["tail_dim"]
    x = np.random.default_rng(2).standard_normal(p.n)
    y = f.solve(x)
    assert np.linalg.norm(f.apply_operator(y) - x) <= 1e-8 * np.linalg.norm(x)
    rep, xs = ce.pcg(a, p.n, p.rhs, f, ce.PcgOptions(tol=p.tol, maxit=200))
    assert rep.converged and rep.iterations <= 3
    assert np.linalg.norm(p.rhs - a.matvec(xs)) <= 10 * p.tol * np.linalg.norm(p.rhs)
    g = ce.ce_factorize(a, p.plan, p.strategy())
    assert np.array_equal(g.solve(x), y)


def test_block_limit_fails_loudly(gpu_ctx):
    """3-D all-axis merges grow blocks with the cell surface: cfg4's stencil at 32^3 reaches
    b ~ 580 at level 3, above the sweep's kSweepBlockMax (256).  The library must refuse with a
    clear error instead of overrunning its shared-memory chunk maps."""
    p = ce.Problem(4, 32, 32, 32, plan="merge_all_axes")
    a = ce.DeviceMatrix(p.matrix())
    with pytest.raises((RuntimeError, ValueError), match="exceeds"):
        ce.ce_factorize(a, p.plan, p.strategy())
    # the context stays usable afterwards
    q = ce.Problem(1, 32, 32)
    b = ce.DeviceMatrix(q.matrix())
    f = ce.ce_factorize(b, q.plan, q.strategy(), ce.FactorOptions(dense_threshold=256))
    rep, _ = ce.pcg(b, q.n, q.rhs, f, ce.PcgOptions(tol=q.tol))
    assert rep.converged
