"""The N>1 bench path (replicas only) on CPU: world_size 2 over
gloo, the time is the max over ranks and the work the sum (bench.reduce_over_ranks)."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import bench
    ms, its = bench.reduce_over_ranks(100.0 + 50.0 * rank, 10 + rank, device="cpu")
    q.put((rank, ms, its))
    dist.destroy_process_group()


def test_reduce_over_ranks_world_size_2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    out = sorted(q.get(timeout=10) for _ in range(2))
    for rank, ms, its in out:
        assert ms == 150.0 and its == 21.0


def test_reduce_single_process_is_identity():
    import bench
    assert bench.reduce_over_ranks(12.5, 7) == (12.5, 7.0)
