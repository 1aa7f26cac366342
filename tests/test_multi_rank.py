"""CPU, world_size 2 over gloo: the multi-GPU sharding path (each rank decodes
its own channel slice, results gathered in input order) and the bench's
max-over-ranks timing helper."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_15685_b200.shard import decode_sharded, shard_range


def test_shard_range_partitions_exactly():
    for n in (0, 1, 7, 8, 1024, 8192):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    assert shard_range(8192, 8, 3) == (3072, 4096)  # C5: 1024 channels per GPU
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def test_decode_sharded_without_process_group():
    out = decode_sharded(list(range(5)), lambda part: [x * 10 for x in part])
    assert out == [0, 10, 20, 30, 40]


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank: int, world: int, port: int, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        seen = []

        def fake_decode(part):  # stands in for decode_batch on this rank's GPU
            seen.extend(part)
            return [f"r{rank}:{x}" for x in part]

        chans = [f"ch{i}" for i in range(11)]
        out = decode_sharded(chans, fake_decode)
        import bench

        t = bench.max_over_ranks(float(rank + 1), world, "cpu")
        q.put((rank, seen, out, t))
    finally:
        dist.destroy_process_group()


def test_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, seen0, out0, t0), (_, seen1, out1, t1) = res
    assert seen0 == [f"ch{i}" for i in range(6)] and seen1 == [f"ch{i}" for i in range(6, 11)]
    expect = [f"r0:ch{i}" for i in range(6)] + [f"r1:ch{i}" for i in range(6, 11)]
    assert out0 == expect and out1 == expect
    assert t0 == t1 == 2.0  # max over ranks
