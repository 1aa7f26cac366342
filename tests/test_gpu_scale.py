"""GPU parity at the benchmarked configurations (BASELINE configs C2-C4).

* G_large (5M states / 20M arcs) against a run of the REFERENCE decoder itself
  (tests/golden/g_large.json, made by tests/golden/make_large_golden.py): the
  bench's C3 channels over two context-switched segments, and C4's dense
  contexts (100-word label-closed and 5% random arcs);
* G_large C3 shape at the bench's launch shape (256-thread CTAs, many
  channels per SM): 16 channels x 4 segments x 125 frames with a context
  switch per segment, every hypothesis against the CPU oracle;
* C4: 5% LABELS and 5% BITSET contexts on G_large, 8 channels each, oracle;
* C2 in full: 64 channels x 500 frames, partial every frame, all channels.

Bar: bit-identical words, costs (f64), frames, kinds, hits; len(store) and
eps_truncations where the reference reports them.  The north-star tolerance
(costs within 1e-4 relative) is asserted as well.
"""

from __future__ import annotations

import hashlib
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from conftest import fx, load_json

pytestmark = pytest.mark.gpu

L = 2000
SEG = 125
COST_RTOL = 1e-4
THREADS = max(1, min(32, os.cpu_count() or 1))


def _digest(csr) -> str:
    h = hashlib.sha256()
    for a, dt in ((csr.row_offsets, np.int64), (csr.ilabels, np.int64), (csr.olabels, np.int64),
                  (csr.next_states, np.int64), (csr.weights, np.float64)):
        h.update(np.ascontiguousarray(a, dtype=dt).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def g_large():
    from paper_2306_15685_b200 import synth

    csr = synth.benchmark_graph(5_000_000, 4, L, seed=421, f32_weights=True)
    pool = synth.unigram_contexts(csr, 20, range(1000, 1256), num_labels=L)
    return csr, pool


@pytest.fixture(scope="module")
def g_large_oracle(g_large):
    from oracle.oracle import OracleGraph

    return OracleGraph.from_csr(g_large[0])


def ctx_index(c: int, seg: int, n_pool: int) -> int:  # bench.py
    return (c * 131 + seg * 17) % n_pool


def _tuples(hyps):
    return [(h.words, h.cost, h.frame, h.kind, h.fallback) for h in hyps]


def _same(got, want, where):
    assert len(got) == len(want), where
    for a, b in zip(got, want):
        assert a.words == b.words, where
        assert (a.kind, a.frame, a.fallback) == (b.kind, b.frame, b.fallback), where
        assert a.cost == pytest.approx(b.cost, rel=COST_RTOL, abs=1e-9), where
        assert a.cost == b.cost, where
        assert a.hits == b.hits, where


def _oracle_segments(og, jobs, cfg):
    """jobs: per channel a list of (scores [T, L], ctx) segments decoded on one
    persistent oracle channel.  Returns per channel per segment (hyps, rc)."""
    from oracle.oracle import OracleChannel, decode_stream

    def one(segs):
        ch = OracleChannel(og)
        return [decode_stream(og, np.asarray(s, dtype=np.float64), ctx, cfg, channel=ch)
                for s, ctx in segs]

    with ThreadPoolExecutor(max_workers=THREADS) as ex:
        return list(ex.map(one, jobs))


@pytest.mark.parametrize("block", ["256", "default"])
def test_g_large_reference_run(g_large, block, exact, monkeypatch):
    """The reference decoder's own output on G_large (5 channels x 2
    context-switched 125-frame segments): hypotheses bit-exact, len(store),
    eps_truncations and utterance counters equal."""
    import paper_2306_15685_b200 as ab
    from paper_2306_15685_b200 import synth

    if block != "default":
        monkeypatch.setenv("AB_BLOCK", block)
    g = load_json("g_large.json")
    csr, pool = g_large
    assert _digest(csr) == g["digest"]
    reg = ab.ContextRegistry({c.id: c for c in pool}, graph_fingerprint="")
    cfg = ab.DecoderConfig(**g["cfg"], exact_counters=exact)
    runs = g["c3"]
    chans = sorted({r["channel"] for r in runs})
    mats = {c: synth.channel_scores(7, c, 2 * SEG, L) for c in chans}
    dev = {c: ab.init_channel(f"c{c}", reg, None, cfg) for c in chans}
    for seg in range(2):
        rs = [r for r in runs if r["segment"] == seg]
        pairs = []
        for r in rs:
            ch = dev[r["channel"]]
            ab.switch_context(ch, reg, r["context"])
            pairs.append((ch, ab.ScoreMatrix(mats[r["channel"]][seg * SEG:(seg + 1) * SEG])))
        res = ab.decode_batch(pairs, csr, reg, cfg)
        for r, got in zip(rs, res):
            where = (r["channel"], seg)
            assert r["error"] is None and got.error is None, (where, got.error)
            want = [(h["words"], fx(h["cost"]), h["frame"], h["kind"], h["fallback"]) for h in r["hyps"]]
            assert _tuples(got.hypotheses) == want, where
            ch = dev[r["channel"]]
            if exact:
                assert len(ch.store) == r["store_len"], where
                assert ch.eps_truncations == r["eps_truncations"], where
            assert ch.utterance_index == r["utterance_index"], where


def test_g_large_dense_contexts_reference_run(g_large, exact):
    """C4's dense contexts on G_large against the reference: a 100-word
    context (5% of arcs, label-closed -> LABELS) and 5% of arcs drawn
    uniformly (not label-closed -> BITSET)."""
    import paper_2306_15685_b200 as ab
    from paper_2306_15685_b200 import _lib, synth

    g = load_json("g_large.json")
    csr, _ = g_large
    cfg = ab.DecoderConfig(**g["cfg"], exact_counters=exact)
    ctxs = {"words100": synth.unigram_contexts(csr, 100, [2000], num_labels=L)[0],
            "arcs5pct": synth.dense_context(csr, 0.05, 2000)}
    modes = {"words100": _lib.AB_CTX_LABELS, "arcs5pct": _lib.AB_CTX_BITSET}
    scores = synth.channel_scores(7, 0, 2 * SEG, L)[:60]
    for r in g["c4"]:
        ctx = ab.BiasingContext(r["name"], ctxs[r["name"]].arc_indices, -2.0)
        assert len(ctx.arc_indices) == r["k"]
        reg = ab.ContextRegistry({ctx.id: ctx}, graph_fingerprint="")
        ch = ab.init_channel(r["name"], reg, ctx.id, cfg)
        res = ab.decode_batch([(ch, ab.ScoreMatrix(scores))], csr, reg, cfg)[0]
        assert res.error is None, res.error
        want = [(h["words"], fx(h["cost"]), h["frame"], h["kind"], h["fallback"]) for h in r["hyps"]]
        assert _tuples(res.hypotheses) == want, r["name"]
        if exact:
            assert len(ch.store) == r["store_len"], r["name"]
        dg = ab.device_graph(csr)
        assert dg.context_mode(dg.context_handle(ctx)) == modes[r["name"]]


def test_g_large_c3_four_segments_at_bench_shape(g_large, g_large_oracle, monkeypatch):
    """C3 at the bench's launch shape (256-thread CTAs): 16 channels x 4
    segments x 125 frames, a context switch from the bench pool at every
    segment boundary (channel 5 unbiased in segment 2), all hypotheses of all
    segments against the oracle run on the same persistent channels."""
    import paper_2306_15685_b200 as ab
    from paper_2306_15685_b200 import synth

    monkeypatch.setenv("AB_BLOCK", "256")
    csr, pool = g_large
    reg = ab.ContextRegistry({c.id: c for c in pool}, graph_fingerprint="")
    cfg = ab.DecoderConfig(beam=13.0, max_active=7000, max_epsilon_expansion=20, partial_every=10)
    n, S = 16, 4
    mats = [synth.channel_scores(7, c, S * SEG, L) for c in range(n)]

    def ctx_of(c, seg):
        return None if (c, seg) == (5, 2) else pool[ctx_index(c, seg, len(pool))]

    chans = [ab.init_channel(f"c{c}", reg, None, cfg) for c in range(n)]
    got = [[None] * S for _ in range(n)]
    for seg in range(S):
        pairs = []
        for c, ch in enumerate(chans):
            x = ctx_of(c, seg)
            ab.switch_context(ch, reg, x.id if x is not None else None)
            pairs.append((ch, ab.ScoreMatrix(mats[c][seg * SEG:(seg + 1) * SEG])))
        res = ab.decode_batch(pairs, csr, reg, cfg)
        for c, r in enumerate(res):
            assert r.error is None, (c, seg, r.error)
            got[c][seg] = r.hypotheses
    jobs = [[(mats[c][s * SEG:(s + 1) * SEG], ctx_of(c, s)) for s in range(S)] for c in range(n)]
    want = _oracle_segments(g_large_oracle, jobs, cfg)
    for c in range(n):
        for s in range(S):
            hyps, rc = want[c][s]
            assert rc == 0
            _same(got[c][s], hyps, f"channel {c} segment {s}")
    assert all(ch.utterance_index == S for ch in chans)


@pytest.mark.parametrize("kind", ["labels", "bitset"])
def test_g_large_c4_dense_at_bench_shape(g_large, g_large_oracle, kind, monkeypatch):
    """C4: 5%-of-arcs contexts on G_large at 256-thread CTAs, 8 channels x
    60 frames, each channel with its own context, against the oracle."""
    import paper_2306_15685_b200 as ab
    from paper_2306_15685_b200 import _lib, synth

    monkeypatch.setenv("AB_BLOCK", "256")
    csr, _ = g_large
    if kind == "labels":
        ctxs = synth.unigram_contexts(csr, 100, range(3000, 3008), num_labels=L)
    else:
        ctxs = [synth.dense_context(csr, 0.05, 3000 + i, ctx_id=f"d{i}") for i in range(8)]
    reg = ab.ContextRegistry({c.id: c for c in ctxs}, graph_fingerprint="")
    cfg = ab.DecoderConfig(beam=13.0, max_active=7000, partial_every=10)
    mats = [synth.channel_scores(17, c, 60, L) for c in range(8)]
    chans = [ab.init_channel(f"d{c}", reg, ctxs[c].id, cfg) for c in range(8)]
    res = ab.decode_batch([(ch, ab.ScoreMatrix(m)) for ch, m in zip(chans, mats)], csr, reg, cfg)
    want = _oracle_segments(g_large_oracle, [[(m, x)] for m, x in zip(mats, ctxs)], cfg)
    dg = ab.device_graph(csr)
    mode = _lib.AB_CTX_LABELS if kind == "labels" else _lib.AB_CTX_BITSET
    for c in range(8):
        assert dg.context_mode(dg.context_handle(ctxs[c])) == mode
        assert res[c].error is None, res[c].error
        hyps, rc = want[c][0]
        assert rc == 0
        _same(res[c].hypotheses, hyps, f"{kind} channel {c}")
        assert res[c].hypotheses[-1].hits > 0


def test_c2_full_all_channels():
    """C2 in full: G_small, 64 channels x 500 frames, each with its own
    20-word context, a partial hypothesis every frame; every channel's 500
    partials and final against the oracle."""
    import paper_2306_15685_b200 as ab
    from oracle.oracle import OracleGraph
    from paper_2306_15685_b200 import synth

    csr = synth.benchmark_graph(10_000, 4, L, seed=421, f32_weights=True)
    cfg = ab.DecoderConfig(beam=13.0, max_active=7000, partial_every=1)
    ctxs = [synth.unigram_context(csr, 20, c, num_labels=L, ctx_id=f"k{c}") for c in range(64)]
    reg = ab.ContextRegistry({c.id: c for c in ctxs}, graph_fingerprint="")
    mats = [synth.channel_scores(7, c, 500, L) for c in range(64)]
    pairs = [(ab.init_channel(f"ch{c}", reg, f"k{c}", cfg), ab.ScoreMatrix(mats[c])) for c in range(64)]
    res = ab.decode_batch(pairs, csr, reg, cfg)
    want = _oracle_segments(OracleGraph.from_csr(csr), [[(m, x)] for m, x in zip(mats, ctxs)], cfg)
    for c in range(64):
        assert res[c].error is None, res[c].error
        hyps, rc = want[c][0]
        assert rc == 0
        assert len(hyps) == 501
        _same(res[c].hypotheses, hyps, f"channel {c}")
