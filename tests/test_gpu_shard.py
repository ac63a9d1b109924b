"""Subdomain-sharded factorization on the GPU (ce_factorize_sharded).

The sharded factorization of a CE_PLAN_SHARDED problem must be BIT-IDENTICAL, on every rank,
to the single-GPU ce_factorize of the same plan (same factor dump bytes): the box interiors are
swept by their owners, the interface rows by every rank, and the exchanges copy bytes.  The
two-rank case runs two processes (gloo: the exchange is staged through host memory) on the one
GPU the test box has -- their kernels never wait on each other, only the host broadcasts do.
"""

import filecmp
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_1603_09133_b200 as ce
from paper_1603_09133_b200 import _lib as L

pytestmark = pytest.mark.gpu

# (3-D grids small enough for a test have no box-interior cells: 2 x 2 x 2 boxes of a 32^3 grid
#  are 4 x 4 x 4 cells at level 1, all within 2 cells of an inner box face)
CASES = [(2, (256, 256, 0), 512), (1, (0, 0, 0), 256), (3, (256, 192, 0), 512)]
IDS = ["cfg2-256", "cfg1-128", "cfg3-256x192"]


class LocalComm:
    """One rank: every broadcast is a no-op (the owner of every box is this rank)."""

    def __init__(self):
        self.rank, self.world, self.error, self.calls = 0, 1, None, 0

        def _b(user, ptr, nbytes, root):
            self.calls += 1
            return 0
        self.fn = L.BcastFn(_b)


@pytest.mark.parametrize("cfg,grid,dth", CASES, ids=IDS)
def test_sharded_one_rank_bit_identical(gpu_ctx, cfg, grid, dth):
    p = ce.Problem(cfg, *grid, plan="sharded")
    a = ce.DeviceMatrix(p.matrix())
    o = ce.FactorOptions(dense_threshold=dth)
    f1 = ce.ce_factorize(a, p.plan, p.strategy(), o)
    comm = LocalComm()
    fs = ce.ce_factorize_sharded(a, p.plan, p.strategy(), p.box_of_block, comm, o)
    d = tempfile.mkdtemp()
    f1.dump(os.path.join(d, "a.bin"))
    fs.dump(os.path.join(d, "b.bin"))
    assert filecmp.cmp(os.path.join(d, "a.bin"), os.path.join(d, "b.bin"), shallow=False)
    st = fs.stats
    assert st["shard_phase1_rows"] > 0 and st["shard_own_rows"] == st["shard_phase1_rows"]
    x = np.random.default_rng(0).standard_normal(p.n)
    assert np.array_equal(f1.solve(x), fs.solve(x))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, cfg, grid, dth, outdir, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        p = ce.Problem(cfg, *grid, plan="sharded")
        a = ce.DeviceMatrix(p.matrix())
        comm = ce.ShardComm(device="cuda:0")
        f = ce.ce_factorize_sharded(a, p.plan, p.strategy(), p.box_of_block, comm, ce.FactorOptions(dense_threshold=dth))
        path = os.path.join(outdir, f"rank{rank}.bin")
        f.dump(path)
        rep, _ = ce.pcg(a, p.n, p.rhs, f, ce.PcgOptions(tol=p.tol))
        st = f.stats
        q.put((rank, "ok", path, rep.iterations, st["shard_own_rows"], st["shard_phase1_rows"], comm.calls, comm.bytes))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, "error", repr(e), 0, 0, 0, 0, 0))


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("cfg,grid,dth", CASES[:3], ids=IDS[:3])
def test_sharded_multi_rank_bit_identical(gpu_ctx, cfg, grid, dth, world):
    p = ce.Problem(cfg, *grid, plan="sharded")
    a = ce.DeviceMatrix(p.matrix())
    f1 = ce.ce_factorize(a, p.plan, p.strategy(), ce.FactorOptions(dense_threshold=dth))
    d = tempfile.mkdtemp()
    ref = os.path.join(d, "single.bin")
    f1.dump(ref)
    its1 = ce.pcg(a, p.n, p.rhs, f1, ce.PcgOptions(tol=p.tol))[0].iterations
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, cfg, grid, dth, d, q), daemon=True) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in procs]
    for pr in procs:
        pr.join(timeout=120)
    own = 0
    for rank, status, path, its, own_rows, p1, calls, nbytes in res:
        assert status == "ok", path
        assert filecmp.cmp(ref, path, shallow=False), f"rank {rank}: sharded factor differs from the single-GPU one"
        assert its == its1
        assert calls > 0 and nbytes > 0
        own += own_rows
        phase1 = p1
    assert own == phase1 > 0  # the ranks' interior rows partition the phase-1 rows
