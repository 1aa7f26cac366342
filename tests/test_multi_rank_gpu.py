"""Multi-GPU path through the drop-in API (decoder.py:523-525):
two ranks (gloo control plane, world size 2) each decode their channel slice
with the real ``decode_batch`` under ``decode_sharded``; the graph goes to the
rank's default device (LOCAL_RANK modulo the visible GPUs - both ranks share
cuda:0 on a one-GPU box) and the gathered hypotheses must equal a single-rank
decode of the whole batch.  Also runs ``bench.py`` under torchrun with two
ranks on one GPU."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batch():
    import paper_2306_15685_b200 as ab
    from paper_2306_15685_b200 import synth

    csr = synth.benchmark_graph(10_000, 4, 2000, seed=421, f32_weights=True)
    ctxs = {f"k{c}": synth.unigram_context(csr, 20, 50 + c, num_labels=2000, ctx_id=f"k{c}")
            for c in range(4)}
    reg = ab.ContextRegistry(ctxs, graph_fingerprint="")
    cfg = ab.DecoderConfig(beam=13.0, max_active=7000, partial_every=10)
    mats = [synth.channel_scores(5, c, 60, 2000) for c in range(11)]
    return ab, csr, reg, cfg, mats


def _run(ab, csr, reg, cfg, mats):
    chans = [ab.init_channel(f"ch{c}", reg, f"k{c % 4}" if c % 3 else None, cfg)
             for c in range(len(mats))]
    return chans, [(ch, ab.ScoreMatrix(m)) for ch, m in zip(chans, mats)]


def _worker(rank: int, world: int, port: int, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), LOCAL_RANK=str(rank),
                      RANK=str(rank), WORLD_SIZE=str(world))
    os.environ.pop("ARCBOOST_DEVICE", None)
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2306_15685_b200 import device as devmod
        from paper_2306_15685_b200.shard import decode_sharded

        ab, csr, reg, cfg, mats = _batch()
        _, pairs = _run(ab, csr, reg, cfg, mats)
        out = decode_sharded(pairs, lambda part: ab.decode_batch(part, csr, reg, cfg))
        dg = ab.device_graph(csr)
        n = __import__("ctypes").c_int32()
        devmod._lib.load().ab_device_count(__import__("ctypes").byref(n))
        q.put((rank, dg.device, n.value,
               [[(h.words, h.cost, h.frame, h.kind, h.hits) for h in r.hypotheses] for r in out],
               [r.error for r in out]))
    finally:
        dist.destroy_process_group()


def test_two_ranks_real_decoder_match_single_rank():
    import torch.multiprocessing as mp

    ab, csr, reg, cfg, mats = _batch()
    _, pairs = _run(ab, csr, reg, cfg, mats)
    single = ab.decode_batch(pairs, csr, reg, cfg)
    want = [[(h.words, h.cost, h.frame, h.kind, h.hits) for h in r.hypotheses] for r in single]
    assert all(r.error is None for r in single)

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in procs), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, dev, n_dev, hyps, errs in res:
        assert dev == rank % n_dev  # LOCAL_RANK picks the device, not a fixed cuda:0
        assert errs == [None] * len(mats)
        assert hyps == want, rank


def test_bench_two_ranks_one_gpu():
    """bench.py under torchrun with world size 2 on one GPU (weak scaling:
    each rank decodes its own channels; max-over-ranks device time)."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
           "--workload", "c2", "--channels", "16", "--frames", "40", "--steps", "1", "--warmup", "1",
           "--no-e2e", "--no-overhead", "--parity-channels", "2", "--cpu-seconds", "1"]
    r = subprocess.run(cmd, cwd=str(ROOT), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["parity_with_gpu"] is True
