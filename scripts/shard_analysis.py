"""Symbolic model of SURVEY §8(e) subdomain sharding for a BASELINE config (host only, no GPU).

Rebuilds each level's block graph from the level-1 CSB pattern and the plan's group
assignments (base(l+1) = coarsen(sq(l)), all groups alive), then reports per level:
  M, close degree, waves of the reference (lexicographic) order's row DAG,
  for P spatial boxes the share of "interior" rows (whole squared-pattern row inside one
  box -- rows that a box's GPU could sweep with no exchange), and the DAG depth of an
  interior-first order (interior rows of all boxes, then the interface rows).
The sweep is bound by its DAG depth (profiles/r1_summary.md), so the model's quantity is
depth, not flops: sharding across GPUs only helps where the interior rows carry the depth.

usage: python scripts/shard_analysis.py [cfg] [nx ny] [boxes per axis ...]
"""
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import paper_1603_09133_b200 as ce  # noqa: E402


def depth(S, rows=None):
    """Longest path of the DAG 'j depends on i < j with S[j, i]' restricted to `rows` (all if None)."""
    S = S.tocsr()
    M = S.shape[0]
    keep = np.ones(M, bool) if rows is None else rows
    w = np.zeros(M, np.int64)
    ip, ix = S.indptr, S.indices
    for j in range(M):
        if not keep[j]:
            continue
        nb = ix[ip[j]:ip[j + 1]]
        nb = nb[(nb < j) & keep[nb]]
        w[j] = (w[nb].max() + 1) if len(nb) else 0
    return int(w[keep].max()) + 1 if keep.any() else 0


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    grid = [int(x) for x in sys.argv[2:4]] if len(sys.argv) > 3 else [0, 0]
    boxes = [int(x) for x in sys.argv[4:]] if len(sys.argv) > 4 else [2, 4, 8]
    import os
    p = ce.Problem(cfg, grid[0], grid[1], 0, plan=os.environ.get("CE_PLAN", "reference"))
    nx = int(round(np.sqrt(p.n))) if grid[0] == 0 else grid[0]
    M = p.m
    rows = np.repeat(np.arange(M), np.diff(p.row_ptr))
    B = sp.csr_matrix((np.ones(len(rows), bool), (rows, p.col_idx)), shape=(M, M))
    first = p.perm[p.offsets[:-1]]
    pos = np.stack([first % nx, first // nx], 1)  # level-1 block -> grid position of its first cell
    print(f"cfg{cfg} n={p.n} M1={M}; boxes per axis {boxes} (P = k^2 boxes)")
    print("lvl      M  close  waves | " + " | ".join(f"P={k * k:3d}: interior  depth(int-first)" for k in boxes))
    for lvl in range(len(p.plan.assigns) + 1):
        S = (B.astype(np.int32) @ B.astype(np.int32)).astype(bool).tocsr()
        deg = int(np.diff(B.indptr).max()) - 1
        line = f"{lvl + 1:3d} {B.shape[0]:6d} {deg:6d} {depth(S):6d} |"
        for k in boxes:
            box = (pos[:, 0] * k // nx) + k * (pos[:, 1] * k // nx)
            Sc = S.tocoo()
            cross = np.zeros(S.shape[0], bool)
            np.logical_or.at(cross, Sc.row, box[Sc.row] != box[Sc.col])
            interior = ~cross
            # interior-first order: interior rows keep their relative order, interface rows after
            order = np.concatenate([np.nonzero(interior)[0], np.nonzero(cross)[0]])
            inv = np.empty_like(order)
            inv[order] = np.arange(len(order))
            Sp = S[order][:, order]
            d = depth(Sp)
            line += f"   {interior.mean():6.1%}  {d:6d}        |"
        print(line)
        if lvl == len(p.plan.assigns):
            break
        a = np.asarray(p.plan.assigns[lvl])
        G = sp.csr_matrix((np.ones(len(a), bool), (np.arange(len(a)), a)), shape=(len(a), int(a.max()) + 1))
        B = (G.T.astype(np.int32) @ S.astype(np.int32) @ G.astype(np.int32)).astype(bool).tocsr()
        # a group's position: its first member's
        firstm = np.full(G.shape[1], -1)
        for b in range(len(a) - 1, -1, -1):
            firstm[a[b]] = b
        pos = pos[firstm]
        if B.shape[0] <= 2048 // max(1, p.block):  # the dense tail takes over (dim <= 2048)
            break


if __name__ == "__main__":
    main()
