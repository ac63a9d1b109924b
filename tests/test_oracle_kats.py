"""Pin the CPU oracle (oracle/) against the reference's known answers.

The reference's own tests are empty stubs (proj/tests/*.cpp hold only
`#include <doctest.h>`), so the known answers come from the reference SPEC
(/root/reference/SPEC.md examples and acceptance criteria, cited per test) and
from numpy/scipy LAPACK cross-checks.  These run on the CPU (no GPU needed).
"""

import numpy as np
import pytest

from _oracle import OProblem, OracleBreakdown, compress, pattern_op


def dense_to_triplets(a):
    r, c = np.nonzero(a)
    return r, c, a[r, c]


# ---- blocksparse ----

def test_from_triplets_tridiagonal_example():
    """3x3 tridiagonal, partition [0,2,3] -> block(0,1) = [[0],[-1]]."""
    a = np.diag([2.0, 2, 2]) + np.diag([-1.0, -1], 1) + np.diag([-1.0, -1], -1)
    p = OProblem.triplets(3, *dense_to_triplets(a), [0, 2, 3])
    off, rp, ci, vp, vals = p.csb()
    assert rp.tolist() == [0, 2, 4] and ci.tolist() == [0, 1, 0, 1]
    assert vals[vp[1]:vp[2]].tolist() == [0.0, -1.0]
    # SPEC.md:66 lower-triangle input with mirror flag -> identical matrix
    lo = np.tril(a)
    q = OProblem.triplets(3, *dense_to_triplets(lo), [0, 2, 3], mirror_lower=True)
    assert np.array_equal(q.dense(), a)


def test_matvec_examples():
    """identity -> x; tridiagonal x ones -> (1, 0, 1)."""
    p = OProblem.triplets(3, [0, 1, 2], [0, 1, 2], [1.0, 1, 1], [0, 1, 2, 3])
    assert p.matvec([1.0, 2, 3]).tolist() == [1, 2, 3]
    a = np.diag([2.0, 2, 2]) + np.diag([-1.0, -1], 1) + np.diag([-1.0, -1], -1)
    q = OProblem.triplets(3, *dense_to_triplets(a), [0, 2, 3])
    assert q.matvec(np.ones(3)).tolist() == [1, 0, 1]


def test_matvec_random_dense():
    """matvec agrees with dense product to 1e-13 relative."""
    rng = np.random.default_rng(1)
    for n in (7, 20, 64):
        b = rng.standard_normal((n, n))
        a = b + b.T
        off = np.unique(np.r_[0, np.sort(rng.choice(np.arange(1, n), size=min(5, n - 1), replace=False)), n])
        p = OProblem.triplets(n, *dense_to_triplets(a), off)
        x = rng.standard_normal(n)
        assert np.linalg.norm(p.matvec(x) - a @ x) <= 1e-13 * np.linalg.norm(a @ x)


def test_asymmetric_input_rejected():
    """asymmetric input without the mirror flag is an error."""
    with pytest.raises(Exception):
        OProblem.triplets(2, [0, 0, 1, 1], [0, 1, 0, 1], [2.0, 1.0, 0.5, 2.0], [0, 1, 2])


def test_pattern_square_examples():
    """SPEC.md:74-76."""
    ident = [[i] for i in range(4)]
    assert pattern_op(0, ident) == ident
    path = [[j for j in (i - 1, i, i + 1) if 0 <= j < 5] for i in range(5)]
    assert pattern_op(0, path) == [[j for j in range(5) if abs(i - j) <= 2] for i in range(5)]
    dense = [[0, 1, 2]] * 3
    assert pattern_op(0, dense) == dense


def test_far_pattern_examples():
    """SPEC.md:84-86."""
    assert pattern_op(1, [[i] for i in range(4)]) == [[] for _ in range(4)]
    path = [[j for j in (i - 1, i, i + 1) if 0 <= j < 5] for i in range(5)]
    assert pattern_op(1, path) == [[j for j in range(5) if abs(i - j) == 2] for i in range(5)]
    assert pattern_op(1, [[0, 1, 2]] * 3) == [[], [], []]


def test_coarsen_pattern_examples():
    """SPEC.md:94-96."""
    assert pattern_op(2, [[i] for i in range(4)], 2, [0, 0, 1, 1]) == [[0], [1]]
    path = [[j for j in (i - 1, i, i + 1) if 0 <= j < 4] for i in range(4)]
    assert pattern_op(2, path, 2, [0, 0, 1, 1]) == [[0, 1], [0, 1]]
    assert pattern_op(2, path, 4, [0, 1, 2, 3]) == path


def test_pattern_properties_random():
    """far/pattern partition of the square, and the square/coarsen relation.

    SPEC.md:120 states coarsen(square(p), g) >= square(coarsen(p, g)); that direction is false
    for general partitions (a group {1, 2} of the paths 0-1, 2-3 links groups of 0 and 3 in the
    coarse square but not in coarsen(square)).  The Boolean relation that holds is <=, tested here."""
    rng = np.random.default_rng(5)
    for _ in range(20):
        m = int(rng.integers(2, 12))
        a = rng.random((m, m)) < 0.25
        a = a | a.T | np.eye(m, dtype=bool)
        rows = [np.nonzero(a[i])[0].tolist() for i in range(m)]
        sq = pattern_op(0, rows)
        far = pattern_op(1, rows)
        for i in range(m):
            assert sorted(set(far[i]) | set(rows[i])) == sq[i]
            assert not (set(far[i]) & set(rows[i]))
        ng = int(rng.integers(1, m + 1))
        assign = np.r_[np.arange(ng), rng.integers(0, ng, size=m - ng)]
        rng.shuffle(assign)
        lhs = pattern_op(2, sq, ng, assign)
        rhs = pattern_op(0, pattern_op(2, rows, ng, assign))
        for g in range(ng):
            assert set(lhs[g]) <= set(rhs[g])
    # the counterexample to the SPEC's direction
    rows = [[0, 1], [0, 1], [2, 3], [2, 3]]
    lhs = pattern_op(2, pattern_op(0, rows), 3, [0, 1, 1, 2])
    rhs = pattern_op(0, pattern_op(2, rows, 3, [0, 1, 1, 2]))
    assert 2 in rhs[0] and 2 not in lhs[0]


# ---- compression (compression.cpp:20-61) ----

def test_compress_empty_and_zero_fill():
    r, u, s = compress(np.zeros((4, 0)))
    assert r == 0 and u is None
    r, u, s = compress(np.zeros((4, 6)))
    assert r == 0 and u is None


def test_compress_exact_rank_two():
    """F = G H with G 8x2, H 2x24, eps=1e-8 -> r = 2."""
    rng = np.random.default_rng(0)
    f = rng.standard_normal((8, 2)) @ rng.standard_normal((2, 24))
    r, u, s = compress(f, eps=1e-8)
    assert r == 2
    assert np.abs(u.T @ u - np.eye(8)).max() <= 1e-12
    e = (u.T @ f)[r:]
    assert np.linalg.norm(e) <= 1e-8 * s[0]


def test_compress_fixed_rank():
    """FixedRank r=4, B=8, full-rank F -> r = 4."""
    rng = np.random.default_rng(1)
    r, u, s = compress(rng.standard_normal((8, 40)), mode=1, rank=4)
    assert r == 4 and u is not None


def test_compress_singular_values_match_lapack():
    rng = np.random.default_rng(2)
    for b, f in [(8, 64), (16, 128), (16, 8), (32, 576), (40, 700)]:
        F = rng.standard_normal((b, f)) * np.logspace(0, -14, b)[:, None]
        r, u, s = compress(F, eps=1e-6)
        ref = np.linalg.svd(F, compute_uv=False)
        assert np.max(np.abs(ref[:len(s)] - s)) <= 1e-14 * ref[0]
        assert r == int(np.sum(ref > 1e-6 * ref[0]))
        # U1 spans the dominant left singular subspace
        ul, _, _ = np.linalg.svd(F)
        p1, p2 = u[:, :r] @ u[:, :r].T, ul[:, :r] @ ul[:, :r].T
        assert np.abs(p1 - p2).max() <= 1e-10


def test_rank_rule_inclusive_threshold():
    """compression.cpp:53: sigma_k <= thr is discarded (inclusive)."""
    u, _ = np.linalg.qr(np.random.default_rng(3).standard_normal((4, 4)))
    v, _ = np.linalg.qr(np.random.default_rng(4).standard_normal((12, 4)))
    s = np.array([1.0, 0.5, 0.25, 0.125])
    F = (u * s) @ v.T
    r, _, sig = compress(F, eps=0.25 / sig_first(F))
    assert r == 2


def sig_first(F):
    return np.linalg.svd(F, compute_uv=False)[0]


# ---- factorization (acceptance criteria 1, 5, 7, 8) ----

def random_spd(n, rng):
    b = rng.standard_normal((n, n))
    return b @ b.T + n * np.eye(n)


def test_dense_fallback_is_cholesky():
    """N <= dense_threshold -> exact dense Cholesky; solve to 1e-12."""
    rng = np.random.default_rng(7)
    a = random_spd(50, rng)
    p = OProblem.triplets(50, *dense_to_triplets(a), [0, 10, 20, 30, 40, 50])
    f = p.factorize(eps=1e-6, dense_threshold=2048)
    assert f.levels == 0 and f.tail_dim == 50
    bvec = rng.standard_normal(50)
    x = f.solve(bvec)
    assert np.linalg.norm(a @ x - bvec) <= 1e-12 * np.linalg.norm(bvec)
    assert np.linalg.norm(f.reconstruct() - a) <= 1e-13 * np.linalg.norm(a)


def test_oracle_equivalence_random_spd():
    """Acceptance criterion 7: random SPD, eps=1e-14 solve ~ dense solve (1e-8);
    r = B (no truncation) reconstructs to 1e-10."""
    rng = np.random.default_rng(11)
    for trial in range(30):
        n = int(rng.integers(20, 120))
        a = random_spd(n, rng) * (rng.random((n, n)) < 0.3)
        a = (a + a.T) / 2 + n * np.eye(n)
        k = int(rng.integers(3, 9))
        off = np.unique(np.r_[0, np.sort(rng.choice(np.arange(1, n), size=k, replace=False)), n])
        p = OProblem.triplets(n, *dense_to_triplets(a), off)
        f = p.factorize(eps=1e-14, dense_threshold=8)
        bvec = rng.standard_normal(n)
        x = f.solve(bvec)
        assert np.linalg.norm(x - np.linalg.solve(a, bvec)) <= 1e-8 * np.linalg.norm(np.linalg.solve(a, bvec))
        bmax = int(np.max(np.diff(off)))
        g = p.factorize(mode=1, rank=bmax, dense_threshold=8)
        assert np.linalg.norm(g.reconstruct() - a) <= 1e-10 * np.linalg.norm(a)


def test_exactness_limit_diffusion_16cube():
    """Acceptance criterion 1: 16^3 diffusion, B=8, eps=1e-12, dense_threshold=512
    -> ||A - Q^T L L^T Q||_F / ||A||_F <= 1e-9."""
    p = OProblem.reference(0, 16, 16, 16, 8)
    f = p.factorize(eps=1e-12, dense_threshold=512)
    a = p.dense()
    assert f.levels >= 1
    assert np.linalg.norm(f.reconstruct() - a) <= 1e-9 * np.linalg.norm(a)


def test_sparsity_accounting_and_invariants():
    """Acceptance criteria 5, 8: #L_1 = 2 #bsp(A); apply_q round trip;
    reconstructed operator symmetric."""
    p = OProblem.reference(0, 8, 8, 8, 8)
    f = p.factorize(eps=1e-6, dense_threshold=64)
    ls = f.level_stats()
    off, rp, ci, vp, vals = p.csb()
    lower = sum(1 for i in range(p.m) for j in ci[rp[i]:rp[i + 1]] if j <= i)
    assert ls[0]["factor_blocks"] == 2 * lower
    assert ls[0]["predicted_edge"] == lower
    x = np.random.default_rng(0).standard_normal(p.n)
    assert np.linalg.norm(f.apply_q_transpose(f.apply_q(x)) - x) <= 1e-13 * np.linalg.norm(x)
    r = f.reconstruct()
    assert np.abs(r - r.T).max() <= 1e-12 * np.abs(r).max()


def test_accuracy_monotone_in_eps():
    """Acceptance criterion 2 (Table 1 trend) at desk scale."""
    p = OProblem.reference(0, 12, 12, 12, 8)
    a = p.dense()
    bvec = np.ones(p.n)
    xs = np.linalg.solve(a, bvec)
    errs, mem = [], []
    for eps in (1e-2, 1e-4, 1e-6):
        f = p.factorize(eps=eps, dense_threshold=256)
        errs.append(np.linalg.norm(f.solve(bvec) - xs) / np.linalg.norm(xs))
        s = f.summary()
        mem.append(s["l_payload_bytes"] + s["q_payload_bytes"] + s["tail_bytes"])
    assert errs[0] > errs[1] > errs[2]
    assert errs[0] / errs[2] >= 1e2
    assert mem[0] < mem[1] < mem[2]


def test_half_elimination_fixed_rank():
    """Acceptance criterion 4: r = B/2 eliminates >= 45% at level 1."""
    p = OProblem.reference(0, 16, 16, 16, 8)
    f = p.factorize(mode=1, rank=4, dense_threshold=512)
    ls = f.level_stats()
    assert ls[0]["eliminated"] >= 0.45 * p.n


def test_breakdown_negated_diagonal():
    """negated diagonal entry -> breakdown at level 1."""
    p = OProblem.reference(0, 4, 4, 4, 8)
    off, rp, ci, vp, vals = p.csb()
    a = p.dense()
    a[0, 0] = -a[0, 0]
    q = OProblem.triplets(p.n, *dense_to_triplets(a), off)
    with pytest.raises(OracleBreakdown) as e:
        q.factorize(eps=1e-6, dense_threshold=8)
    assert e.value.level == 1 and e.value.block == 0


def test_minres_and_pcg_examples():
    """SPEC.md:371 (A = I converges in one iteration) and preconditioned counts (criterion 3)."""
    p = OProblem.triplets(5, range(5), range(5), [1.0] * 5, [0, 5])
    b = np.arange(1.0, 6.0)
    rep, x = p.krylov(b, None, "minres", tol=1e-12)
    assert rep["iterations"] == 1 and np.allclose(x, b)
    rep, x = p.krylov(b, None, "pcg", tol=1e-12)
    assert rep["iterations"] == 1 and np.allclose(x, b)
    q = OProblem.reference(0, 16, 16, 16, 8)
    f = q.factorize(eps=1e-3, dense_threshold=512)
    rep, _ = q.krylov(np.ones(q.n) / 289.0, f, "minres", tol=1e-10)
    assert rep["converged"] and rep["iterations"] <= 10
    rep0, _ = q.krylov(np.ones(q.n) / 289.0, None, "minres", tol=1e-10, maxit=2000)
    assert rep0["iterations"] >= 50


def test_svd_roundoff_columns_do_not_overflow():
    """Regression: a far-fill concatenation from the oracle's own run (cfg1, colour-major plan,
    level 4, row 18; 39 x 174 with 3 nonzero columns, tests/golden/F_roundoff_tail_cfg1_colored_L4.npy)
    whose QR leaves columns of norm ~1e-155.  The unscaled Householder tau = 2 / v^T v overflowed
    there and every singular value came out NaN (rank = b).  With the scaled reflector and
    Eigen's no-reflection rule for tails <= DBL_MIN: rank 3, sigma equal to LAPACK's."""
    import os
    F = np.load(os.path.join(os.path.dirname(__file__), "golden", "F_roundoff_tail_cfg1_colored_L4.npy"))
    r, basis, sigma = compress(F, eps=1e-4)
    sigma = np.asarray(sigma)
    ref = np.linalg.svd(F, compute_uv=False)
    assert np.all(np.isfinite(sigma))
    assert r == 3
    assert np.max(np.abs(sigma[:3] - ref[:3])) <= 1e-13 * ref[0]
    assert np.all(sigma[3:] <= 1e-12 * ref[0])
