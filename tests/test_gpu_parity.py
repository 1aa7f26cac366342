"""GPU parity: the CUDA path (through the package API / C ABI) against the
reference's golden fixtures and the CPU oracle on identical inputs.

Bar (BASELINE.json north_star): identical words and boosted-arc hits, costs
within 1e-4 relative.  Costs accumulate in f64 in the reference's operation
order, so the tests below require bit-identical costs (a stricter bar).
"""

import numpy as np
import pytest

from conftest import case_inputs, expect_hyps, fx, load_json

pytestmark = pytest.mark.gpu

COST_RTOL = 1e-4  # north-star tolerance; asserted in addition to bit equality


def _decode(csr, scores, ctx, cfg, ch_id="c"):
    import paper_2306_15685_b200 as ab

    reg = None
    if ctx is not None:
        reg = ab.ContextRegistry({ctx.id: ctx}, graph_fingerprint="")
    ch = ab.init_channel(ch_id, reg, ctx.id if ctx is not None else None, cfg)
    res = ab.decode_batch([(ch, ab.ScoreMatrix(scores))], csr, reg, cfg)[0]
    return res, ch


def _oracle(csr, scores, ctx, cfg):
    from oracle.oracle import OracleChannel, OracleGraph, decode_stream

    og = OracleGraph.from_csr(csr)
    ch = OracleChannel(og)
    hyps, rc = decode_stream(og, np.asarray(scores, dtype=np.float64), ctx, cfg, channel=ch)
    return hyps, rc, ch.info()


def _same(got, want, where=""):
    assert len(got) == len(want), where
    for a, b in zip(got, want):
        assert a.words == b.words, where
        assert a.kind == b.kind and a.frame == b.frame and a.fallback == b.fallback, where
        assert a.cost == pytest.approx(b.cost, rel=COST_RTOL, abs=1e-9), where
        assert a.cost == b.cost, where  # bit-exact f64
        assert a.hits == b.hits, where


def test_small_cases_match_reference(small_cases, exact):
    """400+ reference-generated instances: ties, epsilon cycles, negative
    weights, max_active binding, epsilon caps, endpointing, dead channels."""
    for c in small_cases:
        csr, scores, ctx, cfg = case_inputs(c, exact)
        res, ch = _decode(csr, scores, ctx, cfg)
        e = c["expect"]
        if e["error"] is not None:
            assert res.error is not None, c["name"]
            assert ("no active tokens" in res.error) == ("no active tokens" in e["error"]), c["name"]
            continue
        assert res.error is None, (c["name"], res.error)
        got = [(h.words, h.cost, h.frame, h.kind, h.fallback) for h in res.hypotheses]
        assert got == expect_hyps(e), c["name"]
        assert ch.utterance_index == e["utterance_index"], c["name"]
        if exact:
            assert ch.eps_truncations == e["eps_truncations"], c["name"]
            assert len(ch.store) == e["store_len"], c["name"]
        hyps, rc, _ = _oracle(csr, scores, ctx, cfg)
        assert [h.hits for h in res.hypotheses] == [h.hits for h in hyps], c["name"]


@pytest.mark.parametrize("variant", ["f32", "f64"])
def test_c1_full_reference_run(variant, exact):
    """C1: G_small, 1 channel x 500 frames, 20-word context, beam 13 - the exact
    run the reference decoded (golden), f32-stored or f64-stored weights."""
    import paper_2306_15685_b200 as ab
    from paper_2306_15685_b200 import synth

    g = load_json("c1_small.json")
    csr = synth.benchmark_graph(10_000, 4, 2000, seed=421, f32_weights=(variant == "f32"))
    ctx = ab.BiasingContext("ctx1", np.array(g["ctx_arcs"], dtype=np.int64), -2.0)
    cfg = ab.DecoderConfig(**g["cfg"], exact_counters=exact)
    scores = np.random.default_rng([7, 0]).uniform(0.0, 6.0, (500, 2000))
    if variant == "f32":
        scores = scores.astype(np.float32)
    res, ch = _decode(csr, scores, ctx, cfg)
    assert res.error is None, res.error
    e = g["runs"][variant]
    got = [(h.words, h.cost, h.frame, h.kind, h.fallback) for h in res.hypotheses]
    assert got == expect_hyps(e)
    if exact:
        assert len(ch.store) == e["store_len"]
    hyps, rc, _ = _oracle(csr, scores, ctx, cfg)
    _same(res.hypotheses, hyps)
    dg = ab.device_graph(csr)
    assert dg.weights_f32 == (variant == "f32")


def test_c2_subset_partials_every_frame():
    """C2 shape: G_small, 64 channels, each with its own 20-word context,
    partial hypotheses every frame (100 frames here; the bench runs 500)."""
    import paper_2306_15685_b200 as ab
    from paper_2306_15685_b200 import synth

    csr = synth.benchmark_graph(10_000, 4, 2000, seed=421, f32_weights=True)
    cfg = ab.DecoderConfig(beam=13.0, max_active=7000, partial_every=1)
    ctxs = {f"k{c}": synth.unigram_context(csr, 20, c, num_labels=2000, ctx_id=f"k{c}")
            for c in range(64)}
    reg = ab.ContextRegistry(ctxs, graph_fingerprint="")
    mats = [synth.channel_scores(11, c, 100, 2000) for c in range(64)]
    pairs = [(ab.init_channel(f"ch{c}", reg, f"k{c}", cfg), ab.ScoreMatrix(mats[c]))
             for c in range(64)]
    res = ab.decode_batch(pairs, csr, reg, cfg)
    for c in range(0, 64, 9):
        assert res[c].error is None
        hyps, rc, _ = _oracle(csr, mats[c], ctxs[f"k{c}"], cfg)
        assert rc == 0
        _same(res[c].hypotheses, hyps, f"channel {c}")


def test_per_frame_token_sets_match_oracle(exact):
    """advance_frame one frame at a time: the surviving token set (states,
    costs, hits) equals the oracle's after every frame, with max_active binding."""
    import paper_2306_15685_b200 as ab
    from paper_2306_15685_b200 import synth
    from oracle.oracle import OracleChannel, OracleGraph

    csr = synth.benchmark_graph(10_000, 4, 2000, seed=421, f32_weights=True)
    ctx = synth.unigram_context(csr, 20, 3, num_labels=2000)
    cfg = ab.DecoderConfig(beam=13.0, max_active=3000, exact_counters=exact)
    og = OracleGraph.from_csr(csr)
    och = OracleChannel(og)
    ch = ab.init_channel("t", None, None, cfg)
    scores = synth.channel_scores(5, 0, 40, 2000)
    for t in range(40):
        ab.advance_frame(ch, scores[t], csr, ctx, cfg)
        och.advance(scores[t].astype(np.float64), ctx, cfg)
        st, co, hi = och.tokens()
        toks = ch.active_tokens()
        assert [x.state for x in toks] == st.tolist(), t
        assert [x.cost for x in toks] == co.tolist(), t
        assert [x.hits for x in toks] == hi.tolist(), t
        info = och.info()
        assert ch.trailing_silence == info["trailing_silence"]
        if exact:
            assert ch.eps_truncations == info["eps_truncations"]
            assert len(ch.store) == info["store_len"]
        if t % 7 == 3:
            p = ab.partial_hypothesis(ch)
            q = och.partial()
            assert p.words == q.words and p.cost == q.cost and p.hits == q.hits
    f = ab.finalize(ch, csr)
    q = och.finalize()
    assert f.words == q.words and f.cost == q.cost and f.fallback == q.fallback


@pytest.mark.parametrize("mode", ["list", "list_global", "bitset", "labels", "auto"])
def test_context_representations_agree(mode):
    """Sparse contexts (shared-memory hash set; a LIST too large for it is
    searched in global memory) and dense ones (HBM bitset by record position)
    give identical decodes; a 5%-dense context is checked against the oracle."""
    import paper_2306_15685_b200 as ab
    from paper_2306_15685_b200 import _lib, synth
    from paper_2306_15685_b200.device import BatchDecoder, DeviceGraph

    csr = synth.benchmark_graph(10_000, 4, 2000, seed=421, f32_weights=True)
    ctx = synth.dense_context(csr, 0.05, 9) if mode == "bitset" else \
        synth.unigram_context(csr, 80 if mode == "list_global" else 20, 9, num_labels=2000)
    if mode == "list_global":
        assert 1365 < len(ctx.arc_indices) <= 2048
    cfg = ab.DecoderConfig(beam=13.0, max_active=7000, partial_every=10)
    scores = synth.channel_scores(3, 1, 60, 2000)
    dg = DeviceGraph(csr)
    want_mode = {"list": _lib.AB_CTX_LIST, "list_global": _lib.AB_CTX_LIST, "bitset": _lib.AB_CTX_BITSET,
                 "labels": _lib.AB_CTX_LABELS, "auto": _lib.AB_CTX_AUTO}[mode]
    h = dg.register_context(ctx.arc_indices, ctx.discount, want_mode)
    # a unigram context is label-closed: AUTO picks the shared-memory label bitmap
    assert dg.context_mode(h) == (_lib.AB_CTX_LABELS if mode == "auto" else want_mode)
    dec = BatchDecoder(dg, 1)
    dec.init_channel(0, h)
    dec.decode([0], [60], [0], np.ascontiguousarray(scores), 2000, cfg, _lib.AB_MODE_STREAM)
    nh, er, hyps, stride, words = dec.results(1)
    assert er[0] == 0
    want, rc, _ = _oracle(csr, scores, ctx, cfg)
    last = []
    got = []
    for q in range(nh[0]):
        x = hyps[q]
        w = last[:x.shared] + words[x.words_off:x.words_off + x.n_words - x.shared].tolist()
        last = w if x.kind == 0 else []
        got.append((w, x.cost, x.hits))
    assert got == [(h.words, h.cost, h.hits) for h in want]


def test_arena_gc_long_utterance():
    """A 600-frame utterance with a small arena forces many in-kernel garbage
    collections; hypotheses and the reference-visible len(store) are unchanged."""
    import paper_2306_15685_b200 as ab
    from paper_2306_15685_b200 import _lib, synth
    from paper_2306_15685_b200.device import BatchDecoder, Capacity, DeviceGraph

    csr = synth.benchmark_graph(10_000, 4, 2000, seed=421, f32_weights=True)
    ctx = synth.unigram_context(csr, 20, 2, num_labels=2000)
    cfg = ab.DecoderConfig(beam=13.0, partial_every=25)
    scores = synth.channel_scores(8, 0, 600, 2000)
    dg = DeviceGraph(csr)
    h = dg.register_context(ctx.arc_indices, ctx.discount)
    dec = BatchDecoder(dg, 2, Capacity(frontier_rows=32768, arena_records=131072))
    dec.init_channels([0, 1], [h, h])
    dec.decode([0, 1], [600, 300], [0, 0], np.ascontiguousarray(scores), 2000, cfg,
               _lib.AB_MODE_STREAM)
    nh, er, hyps, stride, words = dec.results(2)
    assert er.tolist() == [0, 0]
    for c, T in ((0, 600), (1, 300)):
        want, rc, info = _oracle(csr, scores[:T], ctx, cfg)
        last, got = [], []
        for q in range(nh[c]):
            x = hyps[c * stride + q]
            w = last[:x.shared] + words[x.words_off:x.words_off + x.n_words - x.shared].tolist()
            last = w if x.kind == 0 else []
            got.append((w, x.cost, x.hits, x.frame))
        assert got == [(h.words, h.cost, h.hits, h.frame) for h in want]


def test_labels_mode_rejected_for_non_closed_context():
    from paper_2306_15685_b200 import _lib, synth
    from paper_2306_15685_b200.device import DeviceGraph

    csr = synth.benchmark_graph(10_000, 4, 2000, seed=421, f32_weights=True)
    ctx = synth.unigram_context(csr, 20, 9, num_labels=2000)
    dg = DeviceGraph(csr)
    with pytest.raises(_lib.AbError):
        dg.register_context(ctx.arc_indices[1:], -2.0, _lib.AB_CTX_LABELS)
    h = dg.register_context(ctx.arc_indices[1:], -2.0)
    assert dg.context_mode(h) == _lib.AB_CTX_LIST


def test_zero_discount_context_is_identity():
    """SPEC zero-discount identity: a 0.0-discount context changes nothing."""
    import paper_2306_15685_b200 as ab
    from paper_2306_15685_b200 import synth

    csr = synth.benchmark_graph(10_000, 4, 2000, seed=421, f32_weights=True)
    ctx = synth.unigram_context(csr, 100, 4, num_labels=2000, discount=0.0)
    cfg = ab.DecoderConfig(beam=13.0)
    scores = synth.channel_scores(2, 0, 50, 2000)
    a, _ = _decode(csr, scores, None, cfg)
    b, _ = _decode(csr, scores, ctx, cfg)
    assert [(h.words, h.cost) for h in a.hypotheses] == [(h.words, h.cost) for h in b.hypotheses]


def test_context_switch_per_segment():
    """C3 shape: 4 utterance segments per channel with a context switch at each
    boundary (harness.py:208-242 waves)."""
    import paper_2306_15685_b200 as ab
    from paper_2306_15685_b200 import synth

    csr = synth.benchmark_graph(10_000, 4, 2000, seed=421, f32_weights=True)
    pool = {f"p{i}": synth.unigram_context(csr, 20, 100 + i, num_labels=2000, ctx_id=f"p{i}")
            for i in range(6)}
    reg = ab.ContextRegistry(pool, graph_fingerprint="")
    from oracle.oracle import OracleChannel, OracleGraph, decode_stream

    cfg = ab.DecoderConfig(beam=13.0, partial_every=10)
    chans = [ab.init_channel(f"c{i}", reg, None, cfg) for i in range(4)]
    og = OracleGraph.from_csr(csr)
    ochans = [OracleChannel(og) for _ in range(4)]  # persist like the device channels
    for seg in range(4):
        pairs = []
        for i, ch in enumerate(chans):
            ab.switch_context(ch, reg, f"p{(i + seg) % 6}")
            pairs.append((ch, ab.ScoreMatrix(synth.channel_scores(40 + seg, i, 25, 2000))))
        res = ab.decode_batch(pairs, csr, reg, cfg)
        for i, r in enumerate(res):
            assert r.error is None
            want, rc = decode_stream(og, pairs[i][1].costs.astype(np.float64),
                                     pool[f"p{(i + seg) % 6}"], cfg, channel=ochans[i])
            assert rc == 0
            _same(r.hypotheses, want, f"seg {seg} ch {i}")
        assert all(ch.utterance_index == seg + 1 for ch in chans)


def test_g_large_subset():
    """C3/C5 graph (5M states / 20M arcs, direct token table): a channel subset
    against the oracle."""
    import paper_2306_15685_b200 as ab
    from paper_2306_15685_b200 import synth

    csr = synth.benchmark_graph(5_000_000, 4, 2000, seed=421, f32_weights=True)
    ctx = synth.unigram_context(csr, 20, 5, num_labels=2000)
    reg = ab.ContextRegistry({ctx.id: ctx}, graph_fingerprint="")
    cfg = ab.DecoderConfig(beam=13.0, max_active=7000, partial_every=10)
    mats = [synth.channel_scores(21, c, 30, 2000) for c in range(3)]
    pairs = [(ab.init_channel(f"g{c}", reg, ctx.id if c != 1 else None, cfg), ab.ScoreMatrix(m))
             for c, m in enumerate(mats)]
    res = ab.decode_batch(pairs, csr, reg, cfg)
    for c in range(3):
        assert res[c].error is None, res[c].error
        want, rc, _ = _oracle(csr, mats[c], ctx if c != 1 else None, cfg)
        _same(res[c].hypotheses, want, f"channel {c}")


def test_margin_suite_on_device():
    """Reference margin suite: biasing flips all 50 entity decisions on the GPU."""
    m = load_json("margin_suite.json")
    base = {"graph": m["graph"], "cfg": m["cfg"]}
    for u in m["utts"]:
        for key, use_ctx in (("unbiased", False), ("biased", True)):
            c = dict(base, scores=u["scores"], ctx=m["ctx"] if use_ctx else None)
            csr, scores, ctx, cfg = case_inputs(c)
            res, _ = _decode(csr, scores, ctx, cfg)
            assert res.error is None
            got = [(h.words, h.cost, h.frame, h.kind, h.fallback) for h in res.hypotheses]
            assert got == expect_hyps(u[key]), (u["utt_id"], key)
        assert res.hypotheses[-1].words == u["transcript"]


def test_hashed_token_table_matches_reference(small_cases, monkeypatch):
    """The hashed token table (graphs whose direct table does not fit the
    memory budget): forced with table_slots < num_states, so linear probing,
    key claims and slot collisions are exercised; same golden fixtures and
    oracle as the direct table."""
    import paper_2306_15685_b200 as ab
    from paper_2306_15685_b200 import device, synth

    n_hashed = 0
    for i, c in enumerate(small_cases[:200]):
        csr, scores, ctx, cfg = case_inputs(c, exact=bool(i % 2))
        if csr.num_states < 3:
            continue
        # fewer slots than states selects the hashed table (rounded up to a power of two)
        monkeypatch.setattr(device, "DEFAULT_CAPACITY", device.Capacity(table_slots=csr.num_states - 1))
        n_hashed += 1
        res, ch = _decode(csr, scores, ctx, cfg)
        e = c["expect"]
        if e["error"] is not None:
            assert res.error is not None, c["name"]
            continue
        assert res.error is None, (c["name"], res.error)
        got = [(h.words, h.cost, h.frame, h.kind, h.fallback) for h in res.hypotheses]
        assert got == expect_hyps(e), c["name"]
        if cfg.exact_counters:
            assert len(ch.store) == e["store_len"], c["name"]
    assert n_hashed > 100
    monkeypatch.setattr(device, "DEFAULT_CAPACITY", device.Capacity(table_slots=16384))
    csr = synth.benchmark_graph(10_000, 4, 2000, seed=421, f32_weights=True)
    ctx = synth.unigram_context(csr, 20, 1, num_labels=2000)
    cfg = ab.DecoderConfig(beam=13.0, max_active=7000, partial_every=5)
    scores = synth.channel_scores(7, 0, 40, 2000)
    res, ch = _decode(csr, scores, ctx, cfg)
    assert res.error is None, res.error
    want, rc, info = _oracle(csr, scores, ctx, cfg)
    assert rc == 0
    _same(res.hypotheses, want, "G_small hashed")


@pytest.mark.parametrize("beam,max_active", [(float("inf"), 500), (0.25, 7000), (13.0, 1)])
def test_extreme_beams_and_caps(beam, max_active, exact):
    """Infinite beam (max_active alone prunes), a beam narrower than the cost
    spread, and max_active = 1: the prune's cost-bucket split stays exact."""
    import paper_2306_15685_b200 as ab
    from paper_2306_15685_b200 import synth

    csr = synth.benchmark_graph(10_000, 4, 2000, seed=421, f32_weights=True)
    ctx = synth.unigram_context(csr, 20, 9, num_labels=2000)
    cfg = ab.DecoderConfig(beam=beam, max_active=max_active, partial_every=7, exact_counters=exact)
    scores = synth.channel_scores(13, 0, 30, 2000)
    res, ch = _decode(csr, scores, ctx, cfg)
    assert res.error is None, res.error
    want, rc, info = _oracle(csr, scores, ctx, cfg)
    assert rc == 0
    _same(res.hypotheses, want, f"beam {beam} max_active {max_active}")
    if exact:
        assert len(ch.store) == info["store_len"]


def test_full_size_launch_shapes_agree(monkeypatch):
    """Race check at C3 scale (5M-state graph, 256 biased channels): 256-,
    512- and 1024-thread CTAs and a short grid (several channels per CTA, in
    a different order) give bit-identical hypotheses — the CAS recombination,
    warp-aggregated row reservation and kill queues leave no trace of
    scheduling — and two channels match the CPU oracle."""
    import gc

    import paper_2306_15685_b200 as ab
    from paper_2306_15685_b200 import synth

    csr = synth.benchmark_graph(5_000_000, 4, 2000, seed=421, f32_weights=True)
    pool = synth.unigram_contexts(csr, 20, range(1000, 1008), num_labels=2000)
    reg = ab.ContextRegistry({c.id: c for c in pool}, graph_fingerprint="")
    cfg = ab.DecoderConfig(beam=13.0, max_active=7000, partial_every=10)
    n, T = 256, 24
    mats = [ab.ScoreMatrix(synth.channel_scores(7, c, T, 2000)) for c in range(n)]

    def run():
        chans = [ab.init_channel(f"f{c}", reg, pool[c % 8].id, cfg) for c in range(n)]
        res = ab.decode_batch(list(zip(chans, mats)), csr, reg, cfg)
        out = [[(h.words, h.cost, h.frame, h.kind, h.hits) for h in r.hypotheses] for r in res]
        assert all(r.error is None for r in res)
        del chans, res
        gc.collect()
        return out

    shapes = [("256", None), ("512", None), ("1024", None), ("256", "37")]
    outs = []
    for block, grid in shapes:
        monkeypatch.setenv("AB_BLOCK", block)
        if grid:
            monkeypatch.setenv("AB_GRID", grid)
        else:
            monkeypatch.delenv("AB_GRID", raising=False)
        outs.append(run())
    for (block, grid), o in zip(shapes[1:], outs[1:]):
        assert o == outs[0], (block, grid)
    for c in (0, 131):
        want, rc, _ = _oracle(csr, mats[c].costs, pool[c % 8], cfg)
        assert rc == 0
        assert [(h.words, h.cost, h.frame, h.kind, h.hits) for h in want] == outs[0][c], c


def test_smem_token_table_matches_global(monkeypatch):
    """Small graphs at 1024 threads keep the token table in shared memory.
    It must give the same hypotheses as the HBM table, and alternating the
    two across calls on the same channels (epoch tags wrapping every 127
    frames in between) must not let a stale tag of either table alias."""
    import gc

    import paper_2306_15685_b200 as ab
    from paper_2306_15685_b200 import synth

    csr = synth.benchmark_graph(10_000, 4, 2000, seed=421, f32_weights=True)
    pool = synth.unigram_contexts(csr, 20, range(1000, 1004), num_labels=2000)
    reg = ab.ContextRegistry({c.id: c for c in pool}, graph_fingerprint="")
    cfg = ab.DecoderConfig(beam=13.0, max_active=7000, partial_every=10)
    n, T = 4, 140
    utts = [[ab.ScoreMatrix(synth.channel_scores(30 + u, c, T, 2000)) for c in range(n)] for u in range(3)]

    def run(modes):
        chans = [ab.init_channel(f"s{c}", reg, pool[c].id, cfg) for c in range(n)]
        out = []
        for u, smem in enumerate(modes):
            if smem:
                monkeypatch.delenv("AB_NO_SMEM_TABLE", raising=False)
            else:
                monkeypatch.setenv("AB_NO_SMEM_TABLE", "1")
            res = ab.decode_batch(list(zip(chans, utts[u])), csr, reg, cfg)
            assert all(r.error is None for r in res)
            out.append([[(h.words, h.cost, h.frame, h.kind, h.hits) for h in r.hypotheses] for r in res])
        del chans
        gc.collect()
        return out

    monkeypatch.setenv("AB_BLOCK", "1024")
    ref = run([False, False, False])
    assert run([True, True, True]) == ref
    assert run([True, False, True]) == ref
    assert run([False, True, False]) == ref
    for c in range(2):
        want, rc, _ = _oracle(csr, utts[0][c].costs, pool[c], cfg)
        assert rc == 0
        assert [(h.words, h.cost, h.frame, h.kind, h.hits) for h in want] == ref[0][c]


def test_cutoff_engages_and_changes_nothing_observable():
    """The expansion-time cutoff (default mode) relaxes far fewer candidates
    than exact_counters, yet every hypothesis, surviving token set and
    trailing-silence count is the same; a margin of zero forces hint misses,
    whose frames are redone unfiltered (still exact)."""
    import dataclasses
    import os

    import paper_2306_15685_b200 as ab
    from paper_2306_15685_b200 import synth

    csr = synth.benchmark_graph(10_000, 4, 2000, seed=421, f32_weights=True)
    ctxs = {f"k{c}": synth.unigram_context(csr, 20, c, num_labels=2000, ctx_id=f"k{c}") for c in range(8)}
    reg = ab.ContextRegistry(ctxs, graph_fingerprint="")
    fast = ab.DecoderConfig(beam=13.0, max_active=2000, partial_every=3)
    mats = [synth.channel_scores(23, c, 80, 2000) for c in range(8)]

    def run(cfg):
        chans = [ab.init_channel(f"x{c}", reg, f"k{c}", cfg) for c in range(8)]
        res = ab.decode_batch([(ch, ab.ScoreMatrix(m)) for ch, m in zip(chans, mats)], csr, reg, cfg)
        return res, chans

    res_f, ch_f = run(fast)
    res_x, ch_x = run(dataclasses.replace(fast, exact_counters=True))
    for a, b in zip(res_f, res_x):
        assert a.error is None and b.error is None
        _same(a.hypotheses, b.hypotheses)
    eps_f = sum(ch.work_counters[2] for ch in ch_f)
    eps_x = sum(ch.work_counters[2] for ch in ch_x)
    assert eps_f < 0.8 * eps_x, (eps_f, eps_x)
    # forced hint misses: every filtered attempt fails verification and is redone
    old = {k: os.environ.get(k) for k in ("AB_CUT_HINT_MIN", "AB_CUT_HINT_EXTRA")}
    try:
        os.environ["AB_CUT_HINT_MIN"] = "0"
        os.environ["AB_CUT_HINT_EXTRA"] = "-3"
        ab._lib.load().ab_reload_env()
        res_m, ch_m = run(fast)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        ab._lib.load().ab_reload_env()
    for a, b in zip(res_m, res_x):
        _same(a.hypotheses, b.hypotheses)
    assert sum(ch._page.get(ch._slot).cut_redos for ch in ch_m) > 0


@pytest.mark.parametrize("cluster", ["1", "2", "4", "8", "16"])
def test_cluster_sizes_agree(cluster, exact, monkeypatch):
    """A channel decoded by a thread-block cluster (table split
    over DSMEM, counters in the leader) gives the oracle's hypotheses and,
    with exact_counters, its len(store) - for every cluster size, with the
    max_active cut binding and hint misses."""
    import paper_2306_15685_b200 as ab
    from paper_2306_15685_b200 import synth

    monkeypatch.setenv("AB_CLUSTER", cluster)
    csr = synth.benchmark_graph(10_000, 4, 2000, seed=421, f32_weights=True)
    ctxs = {f"q{c}": synth.unigram_context(csr, 20, 40 + c, num_labels=2000, ctx_id=f"q{c}") for c in range(6)}
    reg = ab.ContextRegistry(ctxs, graph_fingerprint="")
    cfg = ab.DecoderConfig(beam=13.0, max_active=2500, partial_every=4, exact_counters=exact)
    mats = [synth.channel_scores(31, c, 50, 2000) for c in range(6)]
    chans = [ab.init_channel(f"k{c}", reg, f"q{c}", cfg) for c in range(6)]
    res = ab.decode_batch([(ch, ab.ScoreMatrix(m)) for ch, m in zip(chans, mats)], csr, reg, cfg)
    for c in range(6):
        assert res[c].error is None, res[c].error
        want, rc, info = _oracle(csr, mats[c], ctxs[f"q{c}"], cfg)
        assert rc == 0
        _same(res[c].hypotheses, want, f"cluster {cluster} channel {c}")
        if exact:
            assert chans[c].eps_truncations == info["eps_truncations"]


@pytest.mark.parametrize("block", ["256", "512"])
def test_small_cases_at_bench_cta_sizes(small_cases, block, monkeypatch):
    """The reference's small cases through the CTA-tile expansion of the
    256 / 512-thread kernels (the bench's C3 shape; small graphs otherwise
    run 1024-thread or cluster kernels), with the cutoff."""
    monkeypatch.setenv("AB_BLOCK", block)
    for c in small_cases[:250]:
        csr, scores, ctx, cfg = case_inputs(c)
        res, ch = _decode(csr, scores, ctx, cfg)
        e = c["expect"]
        if e["error"] is not None:
            assert res.error is not None, c["name"]
            continue
        assert res.error is None, (c["name"], res.error)
        got = [(h.words, h.cost, h.frame, h.kind, h.fallback) for h in res.hypotheses]
        assert got == expect_hyps(e), c["name"]
