"""Full-size oracle fixtures for the GPU parity tests (tests/test_gpu_fullsize_parity.py).

TEST INFRASTRUCTURE ONLY: runs the CPU oracle (oracle/liboracle.so, the
restatement of /root/reference/proj) on a whole BASELINE config and stores a
compact, size-independent summary of its factorization under tests/golden/:

* per level: block sizes, retained ranks and far widths of every row (the
  structure, and the ranks the GPU run is forced to for the re-synchronised
  comparison), LevelStats and the FactorStats summary;
* singular values of sampled rows per level (all level-1 rows' sigma_1);
* operator probes for two seeded vectors x_k: solve(x_k) (= CEFactorization::solve,
  proj/src/factorization.cpp:140-168) and apply_operator(x_k)
  (factorization.cpp:209-257), as sampled entries, the 2-norm and projections on
  four seeded vectors;
* PCG on the config's right-hand side (iterations, true residual).

Modes: `free` (the oracle as is), `perturbed` (A's symmetric entries scaled by
1 + 1e-16 z: the oracle's own sensitivity, the "probe" of DESIGN.md §3) and
`forced` (perturbed A, ranks forced to the free run's: the probe for the
rank-forced comparison).

usage: python scripts/make_fullsize_fixture.py CFG PLAN MODE [nx ny nz]
"""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import _oracle as O  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
EPS = {1: 1e-4, 2: 1e-6, 3: 1e-6, 4: 1e-5, 5: 1e-4}
TOL = {1: 1e-8, 2: 1e-10, 3: 1e-8, 4: 1e-8, 5: 1e-6}
N_SAMPLE = 4096
N_PROJ = 4
N_X = 2


def probe_vectors(n):
    """The seeded probe inputs; the GPU test regenerates them identically."""
    xs = [np.random.default_rng(100 + k).standard_normal(n) for k in range(N_X)]
    ys = [np.random.default_rng(200 + j).standard_normal(n) for j in range(N_PROJ)]
    idx = np.sort(np.random.default_rng(300).choice(n, size=min(N_SAMPLE, n), replace=False))
    return xs, ys, idx


def summarize_vec(v, ys, idx):
    return v[idx].copy(), float(np.linalg.norm(v)), np.array([float(v @ y) for y in ys])


def fixture_name(cfg, plan, mode, grid):
    g = "" if not any(grid) else "_" + "x".join(str(x) for x in grid if x)
    return os.path.join(GOLDEN, f"fullsize_cfg{cfg}{g}_{plan}_{mode}.npz")


def main():
    cfg, plan, mode = int(sys.argv[1]), sys.argv[2], sys.argv[3]
    grid = tuple(int(a) for a in sys.argv[4:7]) if len(sys.argv) > 4 else (0, 0, 0)
    prob = O.OProblem.config(cfg, *grid, plan=plan)
    n = prob.n
    forced = None
    if mode in ("perturbed", "forced"):
        O.lib.oracle_problem_perturb(prob.h, 1e-16, 5)
    if mode == "forced":
        free = np.load(fixture_name(cfg, plan, "free", grid))
        cnt = free["level_m"]
        flat = free["retained"]
        forced, at = [], 0
        for m in cnt:
            forced.append(flat[at:at + m].astype(np.int64).tolist())
            at += m
    t0 = time.time()
    f = prob.factorize(eps=EPS[cfg], forced=forced)
    fac_s = time.time() - t0
    out = dict(cfg=cfg, plan=plan, mode=mode, n=n, eps=EPS[cfg], tol=TOL[cfg], factor_seconds=fac_s,
               tail_dim=f.tail_dim)
    sizes, rets, fcs, ms = [], [], [], []
    sig_rows, sig_lvl, sig_vals, sig_cnt = [], [], [], []
    for lvl in range(f.levels):
        s, r, fc = f.level_structure(lvl)
        sizes.append(s), rets.append(r), fcs.append(fc), ms.append(len(s))
        m = len(s)
        rows = np.arange(m) if lvl == 0 else np.sort(np.random.default_rng(400 + lvl).choice(m, min(256, m), False))
        for b in rows:
            sv = f.row_sigma(lvl, int(b))
            if lvl == 0 and b % 64 and len(sv):
                sv = sv[:1]  # level 1: sigma_1 of every row, the whole spectrum of every 64th
            sig_lvl.append(lvl), sig_rows.append(int(b)), sig_cnt.append(len(sv)), sig_vals.append(sv)
    xs, ys, idx = probe_vectors(n)
    probes = {}
    t1 = time.time()
    for k, x in enumerate(xs):
        for name, fn in (("solve", f.solve), ("op", f.apply_operator)):
            e, nrm, pj = summarize_vec(fn(x), ys, idx)
            probes[f"{name}{k}_samples"], probes[f"{name}{k}_norm"], probes[f"{name}{k}_proj"] = e, nrm, pj
    apply_s = (time.time() - t1) / (2 * N_X)
    rep, xsol = prob.krylov(prob.rhs(), f, method="pcg", tol=TOL[cfg], maxit=1000)
    ls = np.array([[d[k] for k in d] for d in f.level_stats()])
    np.savez_compressed(
        fixture_name(cfg, plan, mode, grid), level_m=np.array(ms, np.int64),
        sizes=np.concatenate(sizes).astype(np.int32), retained=np.concatenate(rets).astype(np.int16),
        fcols=np.concatenate(fcs).astype(np.int32), level_stats=ls,
        summary=np.array(list(f.summary().values())), sample_idx=idx,
        sigma_level=np.array(sig_lvl, np.int16), sigma_row=np.array(sig_rows, np.int32),
        sigma_count=np.array(sig_cnt, np.int32),
        sigma_vals=np.concatenate(sig_vals) if sig_vals else np.zeros(0),
        pcg_iterations=rep["iterations"], pcg_true_resid=rep["true_resid"], pcg_seconds=rep["seconds"],
        meta=json.dumps(dict(out, apply_seconds=apply_s)), **probes)
    print(json.dumps(dict(out, levels=f.levels, apply_seconds=apply_s, pcg=rep)), flush=True)


if __name__ == "__main__":
    main()
