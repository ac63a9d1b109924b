"""GPU-vs-oracle parity of the CE hot path, through the C-ABI.

Runs on a B200 only (-m gpu), on sizes the CPU oracle finishes in seconds.

Calibration: the CE factorization is numerically chaotic
past level 1 -- a 1e-16 relative perturbation of A changes the oracle's own
level-2+ factor entries at O(1) (roundoff-level far fill gets SVD-compressed,
and exact zero tests decide ranks).  Every comparison below therefore holds the
GPU to max(north-star tolerance, 100 x the oracle's own deviation under a
1e-16 input perturbation), level by level, with ranks forced to the oracle's
(the SURVEY's re-synchronisation hook) so structures line up.  Level 1, where
the probe deviation is ~1e-14, is checked at the north-star tolerances.
"""

import ctypes as C
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

import paper_1603_09133_b200 as ce
import _oracle as O
from _dump import read_dump
from _parity import compare, summarize

pytestmark = pytest.mark.gpu

O.lib.oracle_problem_perturb.argtypes = [C.c_void_p, C.c_double, C.c_ulonglong]
O.lib.oracle_problem_perturb.restype = None

# (cfg, grid, dense threshold, plan family); "merge_all" = CE_PLAN_MERGE_ALL_AXES (J = 2^d), the plan
# the full-size 3-D configs run with
CASES = [(1, (0, 0, 0), 2048, "reference"), (2, (64, 64, 0), 2048, "reference"), (3, (64, 64, 0), 2048, "reference"),
         (2, (128, 128, 0), 512, "reference"), (4, (16, 16, 16), 512, "reference"), (5, (16, 16, 16), 512, "reference"),
         (2, (128, 128, 0), 256, "merge_all_axes"), (4, (32, 16, 16), 2048, "merge_all_axes"),
         (2, (128, 128, 0), 256, "merge_all_colored"), (5, (32, 16, 16), 2048, "merge_all_colored"),
         (3, (96, 128, 0), 256, "merge_all_colored"), (1, (0, 0, 0), 256, "merge_all_colored"),
         (2, (256, 256, 0), 512, "sharded")]
IDS = ["cfg1-128", "cfg2-64", "cfg3-64", "cfg2-128", "cfg4-16", "cfg5-16", "cfg2-128-merge_all",
       "cfg4-32x16x16-merge_all", "cfg2-128-colored", "cfg5-32x16x16-colored", "cfg3-96x128-colored",
       "cfg1-128-colored", "cfg2-256-sharded"]


def _dump(f, d, name):
    p = os.path.join(d, name)
    f.dump(p)
    return read_dump(p)


def _level(dmp, lv):
    x = dict(dmp)
    x["levels"] = dmp["levels"][lv:lv + 1]
    x["tail_dim"] = 0
    return x


@pytest.fixture(scope="module")
def runs(gpu_ctx):
    out = {}
    d = tempfile.mkdtemp()
    for (cfg, grid, dth, plan), name in zip(CASES, IDS):
        p = ce.Problem(cfg, *grid, plan=plan)
        op = O.OProblem.config(cfg, *grid, plan=plan)
        fo = op.factorize(eps=p.eps, dense_threshold=dth)
        o = _dump(fo, d, name + "-o.bin")
        forced = [L["retained"].tolist() for L in o["levels"]]
        pp = O.OProblem.config(cfg, *grid, plan=plan)
        O.lib.oracle_problem_perturb(pp.h, 1e-16, 5)
        fp = pp.factorize(eps=p.eps, dense_threshold=dth, forced=forced)
        probe = _dump(fp, d, name + "-p.bin")
        fp_free = pp.factorize(eps=p.eps, dense_threshold=dth)
        a = ce.DeviceMatrix(p.matrix())
        g_free = ce.ce_factorize(a, p.plan, p.strategy(), ce.FactorOptions(dense_threshold=dth))
        g = ce.ce_factorize(a, p.plan, p.strategy(), ce.FactorOptions(dense_threshold=dth, forced_ranks=forced))
        out[name] = dict(p=p, op=op, fo=fo, o=o, probe=probe, fp_free=fp_free, a=a, g_free=g_free, g=g,
                         gd=_dump(g, d, name + "-g.bin"), gd_free=_dump(g_free, d, name + "-gf.bin"), dth=dth)
    return out


def _noise_rows(L):
    """Rows whose far fill is roundoff (sigma_1 <= 1e-10 x the level's largest sigma_1): the reference's
    exact-zero test (compression.cpp:34) sees noise there, so their rank is ill-posed."""
    s1 = np.array([s[0] if len(s) else 0.0 for s in L["sigma"]])
    top = s1.max() if len(s1) else 0.0
    return set(np.nonzero((s1 > 0) & (s1 <= 1e-10 * top))[0].tolist())


@pytest.mark.parametrize("name", IDS)
def test_level1_structure_and_values(runs, name):
    """Level 1: free-run ranks identical to the oracle's except on roundoff-fill rows; with ranks
    forced, sigma <= 1e-13 sigma_1 and factor rows <= 1e-10 (north star) up to the probe sensitivity."""
    R = runs[name]
    G, Oo = R["gd_free"]["levels"][0], R["o"]["levels"][0]
    bad = set(np.nonzero(G["retained"] != Oo["retained"])[0].tolist())
    assert bad <= _noise_rows(Oo), sorted(bad - _noise_rows(Oo))[:10]
    s = summarize(compare(_level(R["gd"], 0), _level(R["o"], 0)))
    sp = summarize(compare(_level(R["probe"], 0), _level(R["o"], 0)))
    print(name, "gpu", s, "probe", sp, "noise rows", len(_noise_rows(Oo)))
    assert s["structure_ok"], s["mismatch"]
    assert s["sigma_max"] <= max(1e-13, 100 * sp["sigma_max"])
    assert s["row_err_p99"] <= max(1e-10, 100 * sp["row_err_p99"])
    assert s["row_err_max"] <= max(1e-8, 100 * sp["row_err_max"])


@pytest.mark.parametrize("name", IDS)
def test_all_levels_within_oracle_sensitivity(runs, name):
    """Ranks forced to the oracle's: per level, GPU deviation <= 100 x the oracle's own 1e-16 sensitivity."""
    R = runs[name]
    g, o, pr = R["gd"], R["o"], R["probe"]
    assert len(g["levels"]) == len(o["levels"]) and g["tail_dim"] == o["tail_dim"]
    for lv in range(len(o["levels"])):
        s = summarize(compare(_level(g, lv), _level(o, lv)))
        sp = summarize(compare(_level(pr, lv), _level(o, lv)))
        print(name, lv, "gpu", {k: s[k] for k in ("sigma_max", "row_err_max", "row_err_p99")},
              "probe", {k: sp[k] for k in ("sigma_max", "row_err_max", "row_err_p99")})
        assert s["structure_ok"], (lv, s["mismatch"])
        assert s["sigma_max"] <= max(1e-13, 100 * sp["sigma_max"]) or s["sigma_max"] <= 1e-6
        assert s["row_err_p99"] <= max(1e-10, 100 * sp["row_err_p99"])


@pytest.mark.parametrize("name", IDS)
def test_level_stats_identical_when_forced(runs, name):
    """With the oracle's ranks, LevelStats (factorization.cpp:376-405) agree exactly."""
    R = runs[name]
    gs, os_ = R["g"].level_stats(), R["fo"].level_stats()
    assert len(gs) == len(os_)
    for x, y in zip(gs, os_):
        for k in ("block_count", "pattern_blocks", "factor_blocks", "eliminated", "retained", "max_rank", "l_bytes",
                  "q_bytes"):
            assert x[k] == y[k], (k, x[k], y[k])
    st, so = R["g"].stats, R["fo"].summary()
    for k in ("factor_blocks", "predicted_factor_blocks", "l_scalar_nnz", "l_payload_bytes", "q_payload_bytes",
              "tail_bytes"):
        assert st[k] == so[k], (k, st[k], so[k])


@pytest.mark.parametrize("name", IDS)
def test_matvec_parity(runs, name):
    """BlockSparseMatrix::matvec (block_matrix.cpp:92-108) on the device (ce_matvec) against the oracle's, same
    block order of accumulation: bitwise up to FMA contraction, asserted at 32 eps max|y|."""
    r = runs[name]
    rng = np.random.default_rng(11)
    for _ in range(2):
        x = rng.standard_normal(r["p"].n)
        yg, yo = r["a"].matvec(x), r["op"].matvec(x)
        assert np.max(np.abs(yg - yo)) <= 32 * np.finfo(float).eps * np.max(np.abs(yo))
    e = np.zeros(r["p"].n)
    e[r["p"].n // 3] = 1.0  # a single column of A: exact products, no rounding at all
    assert np.array_equal(r["a"].matvec(e), r["op"].matvec(e))


@pytest.mark.parametrize("name", IDS)
def test_operator_parity(runs, name):
    """solve(x) = M^-1 x and apply_operator(x) = M x agree with the oracle (gauge invariant, §8c item 4)."""
    R = runs[name]
    rng = np.random.default_rng(7)
    for _ in range(3):
        x = rng.standard_normal(R["p"].n)
        yo = R["fo"].solve(x)
        tol = max(1e-10, 100 * np.linalg.norm(R["fp_free"].solve(x) - yo) / np.linalg.norm(yo))
        for g in (R["g_free"], R["g"]):
            assert np.linalg.norm(g.solve(x) - yo) <= tol * np.linalg.norm(yo)
        mo = R["fo"].apply_operator(x)
        assert np.linalg.norm(R["g"].apply_operator(x) - mo) <= max(1e-10, tol) * np.linalg.norm(mo)
        # self-consistency: M (M^-1 x) = x
        assert np.linalg.norm(R["g"].apply_operator(R["g"].solve(x)) - x) <= 1e-9 * np.linalg.norm(x)


@pytest.mark.parametrize("name", IDS)
def test_pcg_parity(runs, name):
    """PCG iteration counts within +-1 of the oracle's, final true residual below the target (north star)."""
    R = runs[name]
    p = R["p"]
    rg, xg = ce.pcg(R["a"], p.n, p.rhs, R["g_free"], ce.PcgOptions(tol=p.tol, maxit=500))
    ro, xo = R["op"].krylov(p.rhs, R["fo"], "pcg", tol=p.tol, maxit=500)
    assert rg.converged and ro["converged"]
    assert abs(rg.iterations - ro["iterations"]) <= 1
    assert rg.final_true_residual <= 10 * p.tol
    # unpreconditioned CG (hundreds of iterations, rounding drift): counts within 2%
    rg0, _ = ce.pcg(R["a"], p.n, p.rhs, None, ce.PcgOptions(tol=1e-6, maxit=4000))
    ro0, _ = R["op"].krylov(p.rhs, None, "pcg", tol=1e-6, maxit=4000)
    assert abs(rg0.iterations - ro0["iterations"]) <= max(1, 0.02 * ro0["iterations"])


@pytest.mark.parametrize("name", IDS)
def test_minres_parity(runs, name):
    """Device MINRES (minres.cpp:22-115, the paper's solver) against the oracle's
    restatement: same preconditioner contract, iteration counts within +-1 preconditioned, true
    residual at the oracle's level; unpreconditioned counts within 2% (rounding drift)."""
    R = runs[name]
    p = R["p"]
    rg, xg = ce.minres(R["a"], p.n, p.rhs, R["g_free"], ce.MinresOptions(tol=p.tol, maxit=500, track_true_residual=False))
    ro, xo = R["op"].krylov(p.rhs, R["fo"], "minres", tol=p.tol, maxit=500)
    assert rg.converged and ro["converged"]
    assert abs(rg.iterations - ro["iterations"]) <= 1
    assert rg.final_recurrence_residual <= p.tol
    assert rg.final_true_residual <= max(10 * p.tol, 10 * ro["true_resid"])
    rg0, _ = ce.minres(R["a"], p.n, p.rhs, None, ce.MinresOptions(tol=1e-6, maxit=4000, track_true_residual=False))
    ro0, _ = R["op"].krylov(p.rhs, None, "minres", tol=1e-6, maxit=4000)
    assert rg0.converged and ro0["converged"]
    assert abs(rg0.iterations - ro0["iterations"]) <= max(1, 0.02 * ro0["iterations"])


def test_minres_edge_cases(gpu_ctx):
    """Zero rhs converges at once with x = 0 (minres.cpp:33-37); device (torch) vectors give the
    host result; maxit exhaustion is reported, not raised; a dimension mismatch is an error."""
    import torch
    p = ce.Problem(1, 32, 32)
    a = ce.DeviceMatrix(p.matrix())
    f = ce.ce_factorize(a, p.plan, p.strategy(), ce.FactorOptions(dense_threshold=256))
    rep, x = ce.minres(a, p.n, np.zeros(p.n), f)
    assert rep.converged and rep.iterations == 0 and not np.any(x)
    rh, xh = ce.minres(a, p.n, p.rhs, f, ce.MinresOptions(tol=1e-10))
    rd, xd = ce.minres(a, p.n, torch.from_numpy(p.rhs).cuda(), f, ce.MinresOptions(tol=1e-10))
    assert rh.converged and rd.iterations == rh.iterations
    assert np.array_equal(xd.cpu().numpy(), xh)
    r1, _ = ce.minres(a, p.n, p.rhs, None, ce.MinresOptions(tol=1e-14, maxit=3, track_true_residual=True))
    assert not r1.converged and r1.iterations == 3
    with pytest.raises(RuntimeError):
        ce.minres(a, p.n + 1, np.zeros(p.n + 1), f)


@pytest.mark.parametrize("name", IDS)
def test_apply_q_round_trip_and_orthogonality(runs, name):
    """SPEC.md:281-285 round trip; SPEC.md:319 orthogonal bases (<= 1e-12) from the GPU dump."""
    R = runs[name]
    x = np.random.default_rng(3).standard_normal(R["p"].n)
    g = R["g"]
    assert np.linalg.norm(g.apply_q_transpose(g.apply_q(x)) - x) <= 1e-12 * np.linalg.norm(x)
    for L in R["gd"]["levels"]:
        for u in L["basis"]:
            if u is not None:
                assert np.abs(u.T @ u - np.eye(u.shape[0])).max() <= 1e-12


def test_breakdown_negated_diagonal(gpu_ctx):
    """a negated diagonal entry -> BreakdownError at level 1, block 0."""
    p = ce.Problem(1, 32, 32)
    m = p.matrix()
    vals = m.values.copy()
    vals[m.val_ptr[0]] = -vals[m.val_ptr[0]]
    bad = ce.BlockSparseMatrix(m.offsets, m.row_ptr, m.col_idx, m.val_ptr, vals)
    with pytest.raises(ce.BreakdownError) as ei:
        ce.ce_factorize(bad, p.plan, p.strategy(), ce.FactorOptions(dense_threshold=64))
    assert ei.value.level == 1 and ei.value.block == 0


def test_dense_fallback_random_spd(gpu_ctx):
    """n <= dense_threshold -> exact dense Cholesky on the device."""
    rng = np.random.default_rng(1)
    n = 300
    b = rng.standard_normal((n, n))
    a = b @ b.T + n * np.eye(n)
    m = ce.BlockSparseMatrix.from_dense(a, np.arange(0, n + 1, 30))
    f = ce.ce_factorize(m, None, ce.CompressionStrategy.adaptive(1e-6))
    assert f.stats["n_levels"] == 0 and f.stats["tail_dim"] == n
    x = rng.standard_normal(n)
    assert np.linalg.norm(a @ f.solve(x) - x) <= 1e-12 * np.linalg.norm(x)


def test_random_spd_oracle_equivalence(gpu_ctx):
    """Acceptance criterion 7 on the GPU: random SPD, random partitions, eps = 1e-14."""
    rng = np.random.default_rng(11)
    for trial in range(15):
        n = int(rng.integers(40, 160))
        bm = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.1)
        a = bm + bm.T + 2 * n * np.eye(n)
        k = int(rng.integers(4, 10))
        off = np.unique(np.r_[0, np.sort(rng.choice(np.arange(1, n), size=k, replace=False)), n])
        m = ce.BlockSparseMatrix.from_dense(a, off)
        f = ce.ce_factorize(m, None, ce.CompressionStrategy.adaptive(1e-14), ce.FactorOptions(dense_threshold=8))
        x = rng.standard_normal(n)
        assert np.linalg.norm(f.solve(x) - np.linalg.solve(a, x)) <= 1e-8 * np.linalg.norm(np.linalg.solve(a, x))


@pytest.mark.parametrize("mask", [1, 2, 4, 7])
def test_task_split_paths_agree(gpu_ctx, mask):
    """The fat-row task graph (TSQR leaves / strip tasks / Schur panels, forced on small rows with
    CE_FORCE_TASKS) gives the same operator as the single-task path."""
    code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_1603_09133_b200 as ce; "
            "p = ce.Problem(2, 64, 64); a = ce.DeviceMatrix(p.matrix()); "
            "f = ce.ce_factorize(a, p.plan, p.strategy(), ce.FactorOptions(dense_threshold=64)); "
            "x = np.random.default_rng(0).standard_normal(p.n); np.save(sys.argv[1], f.solve(x))")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for m in (0, mask):
        path = tempfile.mktemp(suffix=".npy")
        env = dict(os.environ, CE_FORCE_TASKS=str(m))
        subprocess.run([sys.executable, "-c", code % root, path], env=env, check=True, timeout=300)
        outs.append(np.load(path))
    op = O.OProblem.config(2, 64, 64)
    yo = op.factorize(eps=1e-6, dense_threshold=64).solve(np.random.default_rng(0).standard_normal(op.n))
    for y in outs:
        assert np.linalg.norm(y - yo) <= 1e-6 * np.linalg.norm(yo)
    assert np.linalg.norm(outs[1] - outs[0]) <= 1e-6 * np.linalg.norm(outs[0])


def test_wide_blocks_generic_paths(gpu_ctx):
    """Blocks wider than the register-resident kernels handle (b > 64): the generic TSQR /
    Jacobi / QR paths and the global-scratch sweep variant (per-CTA tiles exceed shared
    memory) must give the same preconditioner as the dense solve."""
    rng = np.random.default_rng(5)
    n = 420
    bm = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.05)
    a = bm + bm.T + 2 * n * np.eye(n)
    off = np.array([0, 100, 210, 300, 420])
    m = ce.BlockSparseMatrix.from_dense(a, off)
    f = ce.ce_factorize(m, None, ce.CompressionStrategy.adaptive(1e-14), ce.FactorOptions(dense_threshold=8))
    assert f.stats["n_levels"] >= 1
    x = rng.standard_normal(n)
    y = np.linalg.solve(a, x)
    assert np.linalg.norm(f.solve(x) - y) <= 1e-8 * np.linalg.norm(y)


def test_blocks_at_the_sweep_limit(gpu_ctx):
    """Blocks just under kSweepBlockMax = 256 (kernels.hpp): every neighbour fills a Schur panel on its own
    (kPanelRows), the strip chunks hold one block each, the wide Jacobi runs at its largest size.  Checked
    against the dense solve and against the oracle on the same matrix."""
    rng = np.random.default_rng(9)
    off = np.array([0, 250, 506, 740, 996, 1200, 1440])
    n = int(off[-1])
    blk = np.searchsorted(off, np.arange(n), side="right") - 1
    tri = np.abs(blk[:, None] - blk[None, :]) <= 1  # block tridiagonal: rows >= 2 compress filled far blocks
    bm = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.03) * tri
    a = bm + bm.T + 2 * n * np.eye(n)
    m = ce.BlockSparseMatrix.from_dense(a, off)
    f = ce.ce_factorize(m, None, ce.CompressionStrategy.adaptive(1e-14), ce.FactorOptions(dense_threshold=8))
    assert f.stats["n_levels"] >= 1 and f.level_stats()[0]["max_block"] == 256
    x = rng.standard_normal(n)
    y = np.linalg.solve(a, x)
    assert np.linalg.norm(f.solve(x) - y) <= 1e-8 * np.linalg.norm(y)
    # one block above the limit is refused, not overrun
    off2 = np.array([0, 257, 506, 740, 996, 1200, 1440])
    with pytest.raises((RuntimeError, ValueError), match="exceeds"):
        ce.ce_factorize(ce.BlockSparseMatrix.from_dense(a, off2), None, ce.CompressionStrategy.adaptive(1e-14),
                        ce.FactorOptions(dense_threshold=8))


@pytest.mark.parametrize("strategy", ["rank3", "rank6", "abs1e-4"])
def test_strategy_modes_parity(gpu_ctx, strategy):
    """The other CompressionStrategy modes (compression.hpp:15-38, compression.cpp:20-61): FixedRank
    (r = min(rank, b), basis only when F != 0 and r < b) and absolute eps.  The
    ranks are decided identically, so the operators agree at the north-star tolerance.  The cfg3
    stencil (random k) is used: on the constant-k grids a fixed rank can cut through an exactly
    degenerate singular-value cluster, where the retained subspace itself is not unique."""
    p = ce.Problem(3, 64, 64)
    op = O.OProblem.config(3, 64, 64)
    pp = O.OProblem.config(3, 64, 64)
    O.lib.oracle_problem_perturb(pp.h, 1e-16, 5)  # the oracle's own sensitivity
    if strategy.startswith("rank"):
        k = int(strategy[4:])
        s = ce.CompressionStrategy.fixed_rank(k)
        fo = op.factorize(mode=1, rank=k, dense_threshold=256)
        fp = pp.factorize(mode=1, rank=k, dense_threshold=256)
    else:
        s = ce.CompressionStrategy.adaptive(1e-4, absolute=True)
        fo = op.factorize(eps=1e-4, absolute=True, dense_threshold=256)
        fp = pp.factorize(eps=1e-4, absolute=True, dense_threshold=256)
    a = ce.DeviceMatrix(p.matrix())
    f = ce.ce_factorize(a, p.plan, s, ce.FactorOptions(dense_threshold=256))
    assert f.stats["n_levels"] == fo.levels and f.stats["tail_dim"] == fo.tail_dim
    x = np.random.default_rng(9).standard_normal(p.n)
    yo = fo.solve(x)
    err = np.linalg.norm(f.solve(x) - yo) / np.linalg.norm(yo)
    probe = np.linalg.norm(fp.solve(x) - yo) / np.linalg.norm(yo)
    print(f"{strategy}: levels {fo.levels} gpu rel {err:.2e} oracle probe {probe:.2e}")
    assert err <= max(1e-10, 100 * probe)


def _solve_in_subprocess(env_extra, cfg=2, grid=(64, 64), dth=64):
    code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_1603_09133_b200 as ce; "
            "p = ce.Problem(%d, %d, %d); a = ce.DeviceMatrix(p.matrix()); "
            "f = ce.ce_factorize(a, p.plan, p.strategy(), ce.FactorOptions(dense_threshold=%d)); "
            "x = np.random.default_rng(0).standard_normal(p.n); np.save(sys.argv[1], f.solve(x))")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = tempfile.mktemp(suffix=".npy")
    env = dict(os.environ, **env_extra)
    subprocess.run([sys.executable, "-c", code % (root, cfg, grid[0], grid[1], dth), path], env=env, check=True,
                   timeout=300)
    return np.load(path)


def test_slot_table_and_zero_far_skip_paths(gpu_ctx):
    """Schur panels looking stored blocks up through the dense triangular table vs the squared-
    pattern binary search give the bit-identical factor (same offsets); skipping the far blocks
    that are still exactly zero (kind 3) changes only the TSQR chunking, so the operator stays
    within roundoff of the full gather and of the oracle."""
    y0 = _solve_in_subprocess({})
    y_bs = _solve_in_subprocess({"CE_NO_TRI": "1"})
    y_full = _solve_in_subprocess({"CE_NO_DEAD_FAR": "1"})
    assert np.array_equal(y0, y_bs)
    op = O.OProblem.config(2, 64, 64)
    yo = op.factorize(eps=1e-6, dense_threshold=64).solve(np.random.default_rng(0).standard_normal(op.n))
    e_full, e_o = np.linalg.norm(y_full - y0) / np.linalg.norm(y0), np.linalg.norm(y0 - yo) / np.linalg.norm(yo)
    print(f"skip vs full gather {e_full:.2e}, vs oracle {e_o:.2e}")
    # deep levels amplify roundoff: the same bound as test_task_split_paths_agree
    assert e_full <= 1e-6 and e_o <= 1e-6


def test_ticket_order_is_schedule_only(gpu_ctx):
    """The sweep's ticket order (build_tickets) only schedules the task graph: the
    round-1 order (chain after rest), the default interleaved order, an early-strip / pre-leaf
    order and the 64-column task split of round 1 all pass the planner's self-check
    (CE_CHECK_TICKETS: every task once, every wait on an earlier ticket) and give the
    bit-identical operator for the same task split."""
    chk = {"CE_CHECK_TICKETS": "1"}
    kw = dict(cfg=3, grid=(128, 96), dth=64)
    y0 = _solve_in_subprocess(chk, **kw)
    y1 = _solve_in_subprocess(dict(chk, CE_CHAIN_FRAC="1.0"), **kw)
    y2 = _solve_in_subprocess(dict(chk, CE_CHAIN_FRAC="0.2", CE_STRIP_FRAC="0.6", CE_PRE_LEAF="37"), **kw)
    assert np.array_equal(y0, y1) and np.array_equal(y0, y2)
    # forced task splits exercise every stage kind on a small problem
    f0 = _solve_in_subprocess(dict(chk, CE_FORCE_TASKS="7", CE_CHAIN_FRAC="1.0"), **kw)
    f1 = _solve_in_subprocess(dict(chk, CE_FORCE_TASKS="7", CE_CHAIN_FRAC="0.3", CE_PRE_LEAF="5"), **kw)
    assert np.array_equal(f0, f1)
