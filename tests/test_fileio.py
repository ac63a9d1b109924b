"""Reference `file` problems through the product library's host loader (ce_problem_load /
ce_problem_save, io.cpp), CPU only: Matrix Market + plan + rhs files as the reference CLI
reads and writes them (proj/src/matrix_market.cpp, problems.cpp:114-182, cli.cpp:49-58,114-150).

The block store the loader builds is pinned to the oracle's restatement of
BlockSparseMatrix::from_triplets (block_matrix.cpp:48-90) on the same triplets; generated
BASELINE problems survive a save -> load round trip bit for bit (%.17g is exact)."""

import os

import numpy as np
import pytest

import paper_1603_09133_b200 as ce
import _oracle as O


def _write_mm(path, n, rows, cols, vals, sym="general", banner=None):
    with open(path, "w") as f:
        f.write(banner or f"%%MatrixMarket matrix coordinate real {sym}\n")
        f.write("% a comment line\n")
        f.write(f"{n} {n} {len(rows)}\n")
        for i, j, v in zip(rows, cols, vals):
            f.write(f"{i + 1} {j + 1} {v:.17g}\n")


def _random_sym(n, density, seed):
    rng = np.random.default_rng(seed)
    a = np.zeros((n, n))
    mask = rng.random((n, n)) < density
    a[mask] = rng.standard_normal(mask.sum())
    a = a + a.T + 2 * n * np.eye(n)
    return a


def _csb(p):
    return p.offsets, p.row_ptr, p.col_idx, p.val_ptr, p.values


def _same(a, b):
    return all(np.array_equal(np.asarray(x), np.asarray(y)) for x, y in zip(a, b))


@pytest.mark.parametrize("plan", ["reference", "merge_all_axes", "merge_all_colored"])
def test_generated_problems_round_trip(tmp_path, plan):
    """run_gen -> load_problem reproduces the CSB, permutation, plan and rhs exactly (every plan
    family travels through the reference's plan-file format)."""
    for cfg, grid in [(1, (32, 32, 0)), (3, (32, 32, 0)), (4, (8, 8, 8))]:
        p = ce.Problem(cfg, *grid, plan=plan)
        m, pl, r = (str(tmp_path / f"{cfg}{s}") for s in ("m.mtx", "plan.txt", "rhs.txt"))
        p.save(m, pl, r)
        q = ce.Problem.load(m, pl, r)
        assert _same(_csb(p), _csb(q))
        assert np.array_equal(p.rhs, q.rhs) and np.array_equal(p.perm, q.perm)
        assert p.plan.join == q.plan.join
        assert len(p.plan.assigns) == len(q.plan.assigns)
        assert all(np.array_equal(a, b) for a, b in zip(p.plan.assigns, q.plan.assigns))
        head = open(m).read(200).splitlines()
        assert head[0] == "%%MatrixMarket matrix coordinate real symmetric"


@pytest.mark.parametrize("sym", ["general", "symmetric"])
def test_loader_matches_oracle_from_triplets(tmp_path, sym):
    """Trivial plan (uniform blocks, identity permutation, ones rhs): the loader's CSB equals the
    oracle's from_triplets CSB, including duplicate summation and ragged last block."""
    n, block = 45, 8
    a = _random_sym(n, 0.08, 1)
    if sym == "general":
        r, c = np.nonzero(a)
        v = a[r, c]
        # split some entries into duplicates (summed on read)
        dup = r[::7].copy(), c[::7].copy(), 0.25 * v[::7]
        v = v.copy()
        v[::7] *= 0.75
        r, c, v = np.concatenate([r, dup[0]]), np.concatenate([c, dup[1]]), np.concatenate([v, dup[2]])
    else:
        r, c = np.nonzero(np.tril(a))
        v = a[r, c]
    path = str(tmp_path / "a.mtx")
    _write_mm(path, n, r, c, v, sym)
    q = ce.Problem.load(path, block=block)
    rr, cc = np.nonzero(a)
    offsets = np.array(list(range(0, n, block)) + [n])
    o = O.OProblem.triplets(n, rr, cc, a[rr, cc], offsets)
    oo = o.csb()
    assert _same(_csb(q)[:4], oo[:4])
    assert np.allclose(_csb(q)[4], oo[4], rtol=0, atol=1e-15 * np.abs(a).max())
    assert np.array_equal(q.rhs, np.ones(n))
    assert np.array_equal(q.perm, np.arange(n)) and len(q.plan.assigns) == 0


def test_loader_with_plan_permutation(tmp_path):
    """A plan file with a permutation, ragged offsets and two levels: the matrix is permuted
    (perm[new] = old) before blocking, like finish_load; checked against the oracle on the
    permuted triplets."""
    n = 30
    rng = np.random.default_rng(2)
    a = _random_sym(n, 0.1, 3)
    perm = rng.permutation(n)
    offsets = [0, 4, 9, 12, 20, 23, 30]
    lv1 = [0, 0, 1, 1, 2, 2]
    lv2 = [0, 1, 0]
    plan = str(tmp_path / "plan.txt")
    with open(plan, "w") as f:
        f.write(f"{n} {len(offsets) - 1} 2 3\n")
        f.write(" ".join(map(str, perm)) + "\n" + " ".join(map(str, offsets)) + "\n")
        f.write(" ".join(map(str, lv1)) + "\n" + " ".join(map(str, lv2)) + "\n")
    rhs = rng.standard_normal(n)
    rpath = str(tmp_path / "rhs.txt")
    np.savetxt(rpath, rhs, fmt="%.17g")
    r, c = np.nonzero(a)
    mpath = str(tmp_path / "a.mtx")
    _write_mm(mpath, n, r, c, a[r, c])
    q = ce.Problem.load(mpath, plan, rpath)
    ap = a[np.ix_(perm, perm)]  # new index p holds old perm[p]
    rr, cc = np.nonzero(ap)
    o = O.OProblem.triplets(n, rr, cc, ap[rr, cc], np.array(offsets))
    assert _same(_csb(q), o.csb())
    assert np.array_equal(q.rhs, rhs[perm])
    assert q.plan.join == 3 and [list(x) for x in q.plan.assigns] == [lv1, lv2]


@pytest.mark.parametrize("case,msg", [
    ("banner", "coordinate real MatrixMarket banner"),
    ("pattern", "coordinate real MatrixMarket banner"),
    ("square", "must be square"),
    ("range", "index out of range"),
    ("truncated", "truncated entry list"),
    ("asym", "asymmetric input"),
    ("plan_perm", "not a bijection"),
    ("plan_group", "empty group"),
    ("plan_dim", "does not match the matrix"),
    ("rhs_len", "rhs length"),
    ("missing", "cannot open"),
])
def test_loader_errors(tmp_path, case, msg):
    """The reference loader's failure modes, each reported as CE_EUSAGE (CLI exit code 1) with its message."""
    n = 4
    a = _random_sym(n, 0.5, 4)
    r, c = np.nonzero(a)
    mpath, plan, rpath = str(tmp_path / "a.mtx"), None, None
    if case == "banner":
        _write_mm(mpath, n, r, c, a[r, c], banner="%%MatrixMarket matrix array real general\n")
    elif case == "pattern":
        _write_mm(mpath, n, r, c, a[r, c], banner="%%MatrixMarket matrix coordinate pattern general\n")
    elif case == "square":
        with open(mpath, "w") as f:
            f.write("%%MatrixMarket matrix coordinate real general\n3 4 1\n1 1 1.0\n")
    elif case == "range":
        _write_mm(mpath, n, list(r) + [n], list(c) + [0], list(a[r, c]) + [1.0])
    elif case == "truncated":
        with open(mpath, "w") as f:
            f.write("%%MatrixMarket matrix coordinate real general\n4 4 3\n1 1 1.0\n")
    elif case == "asym":
        b = a.copy()
        b[0, 1] += 1e-3
        rr, cc = np.nonzero(b)
        _write_mm(mpath, n, rr, cc, b[rr, cc])
    else:
        _write_mm(mpath, n, r, c, a[r, c])
    if case.startswith("plan"):
        plan = str(tmp_path / "plan.txt")
        perm = {"plan_perm": "0 1 1 3", "plan_group": "0 1 2 3", "plan_dim": "0 1 2"}[case]
        offs = "0 2 4" if case != "plan_dim" else "0 1 3"
        lv = "0 2" if case == "plan_group" else "0 0"
        nn = 3 if case == "plan_dim" else n
        with open(plan, "w") as f:
            f.write(f"{nn} 2 1 2\n{perm}\n{offs}\n{lv}\n")
    if case == "rhs_len":
        rpath = str(tmp_path / "rhs.txt")
        np.savetxt(rpath, np.ones(n + 1))
    if case == "missing":
        mpath = str(tmp_path / "nope.mtx")
    with pytest.raises(RuntimeError, match=msg):
        ce.Problem.load(mpath, plan, rpath, block=2)


@pytest.mark.gpu
def test_file_problem_factorizes_like_generated(gpu_ctx, tmp_path):
    """A generated problem written to files and loaded back factorizes to the identical
    preconditioner (bitwise: same inputs, deterministic device factorization)."""
    p = ce.Problem(2, 64, 64)
    fs = [str(tmp_path / s) for s in ("m.mtx", "plan.txt", "rhs.txt")]
    p.save(*fs)
    q = ce.Problem.load(*fs)
    x = np.random.default_rng(5).standard_normal(p.n)
    ys = []
    for prob in (p, q):
        a = ce.DeviceMatrix(prob.matrix())
        f = ce.ce_factorize(a, prob.plan, p.strategy(), ce.FactorOptions(dense_threshold=512))
        ys.append(f.solve(x))
        rep, _ = ce.pcg(a, prob.n, prob.rhs, f, ce.PcgOptions(tol=p.tol))
        assert rep.converged
    assert np.array_equal(ys[0], ys[1])
