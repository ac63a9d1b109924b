"""Host side of the subdomain-sharded factorization, without a GPU.

* CE_PLAN_SHARDED: the product generator and the oracle build the identical plan; every level
  starts with its box-interior rows, box by box (the driver's symbolic split agrees with the
  generator's geometry), and the split over 1/2/4/8 ranks partitions the interior rows;
* ShardComm, the torch.distributed plumbing behind ce_bcast_fn, in a world_size-2 gloo job:
  the in-place broadcast the library issues reaches the other rank.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_1603_09133_b200 as ce
from _oracle import OProblem


@pytest.mark.parametrize("cfg,grid", [(2, (128, 128, 0)), (1, (0, 0, 0)), (3, (96, 128, 0)), (5, (32, 16, 16))])
def test_sharded_plan_matches_oracle(cfg, grid):
    p = ce.Problem(cfg, *grid, plan="sharded")
    o = OProblem.config(cfg, *grid, plan="sharded")
    off, rp, ci, vp, vals = o.csb()
    assert np.array_equal(off, p.offsets) and np.array_equal(rp, p.row_ptr) and np.array_equal(ci, p.col_idx)
    assert np.array_equal(vals, p.values) and np.array_equal(o.perm(), p.perm)
    assigns, join = o.plan_assigns()
    assert len(assigns) == len(p.plan.assigns)
    for x, y in zip(assigns, p.plan.assigns):
        assert np.array_equal(x, y)
    assert p.n_boxes == 8 and p.box_of_block.shape == (p.m,) and set(np.unique(p.box_of_block)) <= set(range(8))


@pytest.mark.parametrize("cfg", [2, 3])
def test_split_partitions_interior_rows(cfg):
    """Full-size cfg2 / cfg3: level 1 is >= 90% box-interior; over every rank count the rows the
    ranks sweep alone partition the interior rows, boxes split evenly between ranks."""
    p = ce.Problem(cfg, plan="sharded")
    base = ce.shard_plan_summary(p, 1)
    assert base[0]["interior"] >= 0.9 * base[0]["blocks"]
    for nr in (2, 4, 8):
        lv = ce.shard_plan_summary(p, nr)
        assert [x["blocks"] for x in lv] == [x["blocks"] for x in base]
        for x in lv:
            assert sum(x["own"]) == x["interior"]
        own1 = lv[0]["own"]
        assert max(own1) - min(own1) <= 0.05 * max(own1)  # balanced boxes


def test_interior_prefix_matches_geometry():
    """The driver's symbolic interior test (every sq(i) label == label(i), as a prefix) finds
    exactly the cells the generator placed first (>= 2 cells inside a box)."""
    p = ce.Problem(2, 256, 256, plan="sharded")
    lv = ce.shard_plan_summary(p, 8)
    # 64 x 64 cells, boxes of 16 x 32 cells: interior = (16-2 or 16-4) x (32-2) per box
    per_box_x = [14, 12, 12, 14]
    assert lv[0]["interior"] == sum(px * 30 for px in per_box_x) * 2
    assert lv[0]["own"] == [px * 30 for px in per_box_x] * 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import ctypes as C
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = ce.ShardComm(device="cpu")
    buf = np.full(1000, float(rank), np.float64)
    if rank == 1:
        buf[:] = np.arange(1000) * 0.5
    rc = comm.fn(None, buf.ctypes.data, buf.nbytes, 1)  # the library's call shape: (user, ptr, bytes, root)
    rc2 = comm.fn(None, buf.ctypes.data_as(C.c_void_p).value + 8 * 10, 8 * 5, 0)
    q.put((rank, rc, rc2, buf.copy(), comm.calls))
    dist.destroy_process_group()


def test_shardcomm_broadcast_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = dict((r, (rc, rc2, b, calls)) for r, rc, rc2, b, calls in (q.get(timeout=120) for _ in procs))
    for pr in procs:
        pr.join(timeout=60)
    expect = np.arange(1000) * 0.5
    expect[10:15] = expect[10:15]  # rank 0's slice after the first broadcast is rank 1's data
    for r in (0, 1):
        rc, rc2, b, calls = out[r]
        assert rc == 0 and rc2 == 0 and calls == 2
        assert np.array_equal(b, expect)
