"""Device assembly (ce_matrix_from_triplets): BlockSparseMatrix::from_triplets
(proj/src/block_matrix.cpp:48-90) on the GPU, bit-identical to the oracle's restatement.

* duplicates summed in input order (random splits of every entry into 1-3 shuffled parts,
  whose left-to-right sum is order dependent in floating point);
* MirrorMode::Lower (one triangle in, both out) and None (both triangles, symmetry checked to
  1e-12 max|a| with the reference's message);
* pattern: every touched block inserted symmetrically + the full diagonal, variable block sizes;
* the BASELINE generator's matrices round-trip through triplets unchanged, and factorize the same.
"""

import numpy as np
import pytest

import paper_1603_09133_b200 as ce
import _oracle as O

pytestmark = pytest.mark.gpu


def _split_shuffle(rows, cols, vals, rng):
    """Each entry as 1-3 parts in random order (duplicates the reference sums in input order)."""
    R, Cc, V = [], [], []
    for r, c, v in zip(rows, cols, vals):
        k = rng.integers(1, 4)
        w = rng.random(k)
        parts = v * w / w.sum()
        for p in parts:
            R.append(r)
            Cc.append(c)
            V.append(p)
    perm = rng.permutation(len(V))
    return np.array(R)[perm], np.array(Cc)[perm], np.array(V)[perm]


def _csb_equal(a, o):
    off, rp, ci, vp, vals = o
    assert np.array_equal(a.offsets, off) and np.array_equal(a.row_ptr, rp) and np.array_equal(a.col_idx, ci)
    assert np.array_equal(a.val_ptr, vp)
    assert np.array_equal(a.values, vals), np.max(np.abs(a.values - vals))  # bit-exact


@pytest.mark.parametrize("mirror", [False, True])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_triplets_bit_identical(gpu_ctx, mirror, seed):
    rng = np.random.default_rng(seed)
    n = 300
    sizes = rng.integers(1, 12, 60)
    sizes = sizes[np.cumsum(sizes) <= n]
    offsets = np.concatenate([[0], np.cumsum(sizes)])
    n = int(offsets[-1])
    a = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.03)
    a = a + a.T + np.diag(rng.random(n) + n)
    r, c = np.nonzero(np.tril(a) if mirror else a)
    v = a[r, c]
    R, Cc, V = _split_shuffle(r, c, v, rng)
    dm = ce.DeviceMatrix.from_triplets(n, R, Cc, V, offsets, mirror_lower=mirror)
    op = O.OProblem.triplets(n, R, Cc, V, offsets, mirror_lower=mirror)
    _csb_equal(dm.csb(), op.csb())
    x = rng.standard_normal(n)
    assert np.allclose(dm.matvec(x), op.matvec(x), rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("cfg,grid", [(1, (0, 0, 0)), (2, (64, 64, 0)), (3, (64, 64, 0)), (4, (16, 16, 16)),
                                      (5, (12, 8, 20))])
def test_generator_csb_round_trip(gpu_ctx, cfg, grid):
    """The generator's CSB as scalar triplets (both triangles, shuffled) -> the identical CSB;
    the factor of the device-assembled matrix equals the uploaded one's."""
    p = ce.Problem(cfg, *grid)
    m = p.matrix()
    R, Cc, V = [], [], []
    bs = np.diff(m.offsets)
    for i in range(m.m):
        for k in range(m.row_ptr[i], m.row_ptr[i + 1]):
            j = m.col_idx[k]
            blk = m.values[m.val_ptr[k]:m.val_ptr[k + 1]].reshape(bs[i], bs[j])
            rr, cc = np.nonzero(np.ones_like(blk))
            R.append(m.offsets[i] + rr)
            Cc.append(m.offsets[j] + cc)
            V.append(blk[rr, cc])
    R, Cc, V = (np.concatenate(x) for x in (R, Cc, V))
    perm = np.random.default_rng(cfg).permutation(len(V))
    dm = ce.DeviceMatrix.from_triplets(p.n, R[perm], Cc[perm], V[perm], m.offsets)
    _csb_equal(dm.csb(), (m.offsets, m.row_ptr, m.col_idx, m.val_ptr, m.values))
    f1 = ce.ce_factorize(dm, p.plan, p.strategy(), ce.FactorOptions(dense_threshold=512))
    f2 = ce.ce_factorize(ce.DeviceMatrix(m), p.plan, p.strategy(), ce.FactorOptions(dense_threshold=512))
    x = np.random.default_rng(5).standard_normal(p.n)
    assert np.array_equal(f1.solve(x), f2.solve(x))


def test_errors_match_reference(gpu_ctx):
    off = np.array([0, 2, 4])
    with pytest.raises(RuntimeError, match="triplet index outside matrix dimension"):
        ce.DeviceMatrix.from_triplets(4, [0, 4], [0, 0], [1.0, 2.0], off)
    R, Cc, V = [0, 1, 2, 3, 0, 2], [0, 1, 2, 3, 2, 0], [4.0, 4.0, 4.0, 4.0, 1.0, 1.5]
    with pytest.raises(RuntimeError) as e:
        ce.DeviceMatrix.from_triplets(4, R, Cc, V, off)
    with pytest.raises(O.OracleError) as eo:
        O.OProblem.triplets(4, R, Cc, V, off)
    assert str(e.value) == str(eo.value) and "asymmetric input" in str(e.value)
