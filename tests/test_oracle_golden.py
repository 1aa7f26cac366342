"""CPU: the oracle (oracle/, test infrastructure) against fixtures produced by
the reference itself (tests/golden/make_golden.py).  This pins the checker the
GPU parity tests rely on."""

import numpy as np
import pytest

from conftest import case_inputs, expect_hyps, fx, load_json

from oracle.oracle import OracleChannel, OracleGraph, decode_stream


def run_oracle(csr, scores, ctx, cfg):
    og = OracleGraph.from_csr(csr)
    ch = OracleChannel(og)
    hyps, rc = decode_stream(og, scores, ctx, cfg, channel=ch)
    return hyps, rc, ch.info()


def test_small_cases_bit_exact(small_cases):
    assert len(small_cases) > 300
    for c in small_cases:
        csr, scores, ctx, cfg = case_inputs(c)
        hyps, rc, info = run_oracle(csr, scores, ctx, cfg)
        e = c["expect"]
        if e["error"] is not None:
            assert rc != 0, c["name"]
            assert ("no active tokens" in e["error"]) == (rc == 1), c["name"]
            continue
        assert rc == 0, c["name"]
        got = [(h.words, h.cost, h.frame, h.kind, h.fallback) for h in hyps]
        assert got == expect_hyps(e), c["name"]
        assert info["utterance_index"] == e["utterance_index"], c["name"]
        assert info["eps_truncations"] == e["eps_truncations"], c["name"]
        assert info["store_len"] == e["store_len"], c["name"]


def test_golden_f1_values(small_cases):
    by = {c["name"]: c for c in small_cases}
    # reference tests/test_decoder.py:86-103
    assert by["f1_easy"]["expect"]["hyps"][-1]["words"] == [1, 2]
    assert fx(by["f1_easy"]["expect"]["hyps"][-1]["cost"]) == pytest.approx(0.8, abs=1e-12)
    assert fx(by["f1_margin_biased"]["expect"]["hyps"][-1]["cost"]) == pytest.approx(-2.2, abs=1e-12)
    assert by["f1_margin"]["expect"]["hyps"][-1]["words"] == [3, 2]


@pytest.mark.parametrize("variant", ["f32", "f64"])
def test_c1_small_oracle_matches_reference(variant):
    from paper_2306_15685_b200 import synth
    import paper_2306_15685_b200 as ab

    g = load_json("c1_small.json")
    csr = synth.benchmark_graph(10_000, 4, 2000, seed=421, f32_weights=(variant == "f32"))
    ctx = ab.BiasingContext("ctx1", np.array(g["ctx_arcs"], dtype=np.int64), -2.0)
    assert np.array_equal(ctx.arc_indices, synth.unigram_context(csr, 20, 1, num_labels=2000).arc_indices)
    cfg = ab.DecoderConfig(**g["cfg"])
    scores = np.random.default_rng([7, 0]).uniform(0.0, 6.0, (500, 2000))
    if variant == "f32":
        scores = scores.astype(np.float32).astype(np.float64)
    hyps, rc, info = run_oracle(csr, scores, ctx, cfg)
    assert rc == 0
    e = g["runs"][variant]
    assert [(h.words, h.cost, h.frame, h.kind, h.fallback) for h in hyps] == expect_hyps(e)
    assert info["store_len"] == e["store_len"]


def test_margin_suite_flips():
    """Reference margin suite (synth.py:218-291): unbiased decodes lose every entity,
    biased decodes recover every one; the oracle reproduces both exactly."""
    import paper_2306_15685_b200 as ab

    m = load_json("margin_suite.json")
    base = {"graph": m["graph"], "ctx": m["ctx"], "cfg": m["cfg"]}
    flips = 0
    for u in m["utts"]:
        for key, use_ctx in (("unbiased", False), ("biased", True)):
            c = dict(base, scores=u["scores"], ctx=m["ctx"] if use_ctx else None)
            csr, scores, ctx, cfg = case_inputs(c)
            hyps, rc, _ = run_oracle(csr, scores, ctx, cfg)
            assert rc == 0
            assert [(h.words, h.cost, h.frame, h.kind, h.fallback) for h in hyps] == expect_hyps(u[key])
        if u["biased"]["hyps"][-1]["words"] == u["transcript"] != u["unbiased"]["hyps"][-1]["words"]:
            flips += 1
    assert flips == 50
