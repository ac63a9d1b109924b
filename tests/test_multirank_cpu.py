"""world_size-2 gloo check of bench.py's multi-rank plumbing (CPU, no GPU):
barrier + max-over-ranks timing and the whole-job throughput formula."""

import os
import socket
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = 1.5 if rank == 0 else 2.5  # per-rank factor time
    dist.barrier()
    tmax = bench.reduce_max(t, dist, "cpu")
    q.put((rank, tmax, bench.job_throughput(world, 1000, 4, tmax)))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_gloo_max_and_throughput():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=100) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [2.5, 2.5]
    assert res[0][2] == pytest.approx(2 * 1000 * 4 / 2.5)


def test_reference_arm_nonzero_rank_exits_clean(monkeypatch):
    import bench
    monkeypatch.setenv("RANK", "1")
    args = type("A", (), dict(cfg=2, grid=[0, 0, 0], steps=1, warmup=0, gpus=2))()
    assert bench.run_reference(args) == 0
