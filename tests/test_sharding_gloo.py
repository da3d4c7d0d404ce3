"""Multi-process (world_size 2, gloo, CPU) test of the stream-sharding and
timing-aggregation path bench.py uses on N GPUs."""
import os
import socket

import pytest

from paper_2308_09209_b200.sharding import stream_assignment


def test_assignment_partitions_streams():
    for n in (1, 7, 64):
        for world in (1, 2, 4, 8):
            got = sorted(s for r in range(world) for s in stream_assignment(n, world, r))
            assert got == list(range(n))
            sizes = [len(stream_assignment(n, world, r)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        stream_assignment(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    from paper_2308_09209_b200 import sharding

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        streams = sharding.stream_assignment(64, world, rank)
        secs = 1.0 + rank  # rank 1 is the slowest
        fps = sharding.aggregate_throughput(len(streams) * 10, secs)
        mx = sharding.max_over_ranks(secs)
        tot = sharding.sum_over_ranks(len(streams))
        dist.barrier()
        q.put((rank, streams, fps, mx, tot))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_aggregate():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    assert out[0][1] == list(range(0, 64, 2)) and out[1][1] == list(range(1, 64, 2))
    for _, _, fps, mx, tot in out:
        assert mx == 2.0  # max over ranks
        assert tot == 64  # every stream served once
        assert fps == pytest.approx(640 / 2.0)  # all frames / slowest rank
