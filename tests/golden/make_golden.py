"""Generate golden fixtures by running the REFERENCE package (read-only import
from /root/reference/pkg/src) on fixed inputs.  Run in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

The reference does not exist on the GPU box, so its outputs travel as these
fixtures.  Floats are stored with float.hex() so parity is checked bit-exactly.

Fixtures:
  small_cases.json     F1/F2 cases of tests/test_decoder.py + 400 random instances
                       (random_fst / random_scores, integer-valued "tie" scores,
                       contexts, pruning, endpointing, epsilon caps)
  c1_small.json        C1: G_small (build_benchmark_graph(10000, 4, 2000, seed=421)),
                       1 channel, 500 frames, 20-word context, beam 13, partial_every 10,
                       for f64 weights and for f32-rounded weights/scores
  graph_digest.json    sha256 of the reference CSR arrays of G_small
  margin_suite.json    build_margin_suite(50): graph, contexts compiled by the
                       reference's Alg. 1, unbiased and biased finals
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from arcboost.biasing import BiasingContext, BoostCompileConfig, ContextRegistry, compile_context  # noqa: E402
from arcboost.decoder import DecoderConfig, decode_batch, init_channel  # noqa: E402
from arcboost.fst import CsrFst, build_csr, parse_text_fst  # noqa: E402
from arcboost.scores import ScoreMatrix  # noqa: E402
from arcboost.synth import build_benchmark_graph, build_margin_suite, random_fst, random_scores  # noqa: E402

OUT = Path(__file__).resolve().parent

F1 = "0 1 1 1 0.5\n0 3 3 3 0.9\n1 2 2 2 0.3\n1 3 0 0 0.1\n3 2 2 2 0.7\n2 0.0\n3 0.4\n"
F2 = "0 1 1 1 0.1\n1 1 2 0 0.0\n1 0.0\n"


def hx(x: float) -> str:
    return float(x).hex()


def graph_json(csr) -> dict:
    return {
        "start": int(csr.start),
        "row_offsets": [int(v) for v in csr.row_offsets],
        "ilabels": [int(v) for v in csr.ilabels],
        "olabels": [int(v) for v in csr.olabels],
        "next_states": [int(v) for v in csr.next_states],
        "weights": [hx(v) for v in csr.weights],
        "finals": [[int(s), hx(w)] for s, w in sorted(csr.finals.items())],
    }


def cfg_json(cfg) -> dict:
    return {"beam": cfg.beam, "max_active": cfg.max_active,
            "max_epsilon_expansion": cfg.max_epsilon_expansion,
            "partial_every": cfg.partial_every,
            "endpoint_silence_frames": cfg.endpoint_silence_frames,
            "silence_ilabel": cfg.silence_ilabel}


def run_ref(csr, scores: np.ndarray, ctx, cfg) -> dict:
    reg = None
    ch = init_channel("c", None, None, cfg)
    if ctx is not None:
        reg = ContextRegistry(contexts={ctx.id: ctx}, graph_fingerprint="")
        ch = init_channel("c", reg, ctx.id, cfg)
    res = decode_batch([(ch, ScoreMatrix(costs=scores))], csr, reg, cfg)[0]
    return {
        "error": res.error,
        "hyps": [{"words": h.words, "cost": hx(h.cost), "frame": h.frame, "kind": h.kind,
                  "fallback": h.fallback} for h in res.hypotheses],
        "store_len": len(ch.store), "utterance_index": ch.utterance_index,
        "eps_truncations": ch.eps_truncations,
    }


def case(name, csr, scores, ctx, cfg) -> dict:
    scores = np.asarray(scores, dtype=np.float64).reshape(len(scores), -1) if len(scores) else \
        np.zeros((0, max(csr.num_emitting_labels, 1)))
    return {
        "name": name,
        "graph": graph_json(csr),
        "scores": [[hx(v) for v in row] for row in scores],
        "width": int(scores.shape[1]),
        "ctx": None if ctx is None else {"arc_indices": [int(v) for v in ctx.arc_indices],
                                         "discount": hx(ctx.discount)},
        "cfg": cfg_json(cfg),
        "expect": run_ref(csr, scores, ctx, cfg),
    }


def small_cases() -> list:
    cases = []
    f1 = build_csr(parse_text_fst(F1))
    f2 = build_csr(parse_text_fst(F2))
    ctx024 = BiasingContext(id="c1", arc_indices=np.array([0, 2, 4]), discount=-2.0)
    easy = [[0.0, 5.0, 5.0], [5.0, 0.0, 5.0]]
    margin = [[1.0, 5.0, 0.0], [5.0, 0.0, 5.0]]
    d = DecoderConfig()
    cases.append(case("f1_easy", f1, easy, None, d))
    cases.append(case("f1_easy_biased", f1, easy, ctx024, d))
    cases.append(case("f1_margin", f1, margin, None, d))
    cases.append(case("f1_margin_biased", f1, margin, ctx024, d))
    cases.append(case("f1_margin_partials", f1, margin, ctx024, DecoderConfig(partial_every=1)))
    cases.append(case("f1_dead", f1, [[0.0, 0.0, 0.0]] * 3, None, DecoderConfig(partial_every=1)))
    cases.append(case("f1_zero_frames", f1, [], None, d))
    cases.append(case("fallback", build_csr(parse_text_fst("0 1 1 1 0.5\n1 2 1 1 0.5\n2 0.0\n")),
                      [[0.0]], None, d))
    cases.append(case("zero_frame_final", build_csr(parse_text_fst("0 1 1 1 0.5\n0 0.25\n1 0.0\n")),
                      [], None, d))
    rows = [[0.0, 5.0]] + [[5.0, 0.0]] * 3 + [[0.0, 5.0]] + [[5.0, 0.0]] * 3
    cases.append(case("f2_endpoint", f2, rows, None,
                      DecoderConfig(silence_ilabel=2, endpoint_silence_frames=3, partial_every=100)))
    cases.append(case("f2_partials3", f2, [[0.0, 0.0]] * 10, None, DecoderConfig(partial_every=3)))
    for seed in range(400):
        rng = random.Random(10_000 + seed)
        fst = random_fst(rng, max_states=rng.choice([4, 12, 30, 60]),
                         max_arcs=rng.choice([10, 40, 120, 240]), num_labels=rng.choice([2, 4, 6]),
                         ensure_emitting=rng.random() < 0.7, all_final=rng.random() < 0.5,
                         eps_input_prob=rng.choice([0.15, 0.4]),
                         weight_range=rng.choice([(0.0, 3.0), (-1.0, 2.0)]))
        csr = build_csr(fst)
        if csr.num_emitting_labels == 0:
            continue
        T = rng.randint(0, 10)
        if rng.random() < 0.4:  # integer scores force cost ties
            sc = [[float(rng.randint(0, 3)) for _ in range(csr.num_emitting_labels)] for _ in range(T)]
        else:
            sc = random_scores(rng, T, csr.num_emitting_labels).costs.tolist()
        ctx = None
        if rng.random() < 0.6 and csr.num_arcs:
            k = rng.randint(1, min(12, csr.num_arcs))
            ctx = BiasingContext(id="r", arc_indices=np.array(sorted(rng.sample(range(csr.num_arcs), k))),
                                 discount=rng.choice([-2.0, -0.5, 0.0, 1.0]))
        cfg = DecoderConfig(beam=rng.choice([1.0, 3.0, 16.0]), max_active=rng.choice([1, 2, 3, 7000]),
                            max_epsilon_expansion=rng.choice([0, 1, 2, 20, 40]),
                            partial_every=rng.choice([1, 2, 10]),
                            endpoint_silence_frames=rng.choice([0, 1, 2, 20]),
                            silence_ilabel=rng.choice([0, 0, 1, 2]))
        cases.append(case(f"random_{seed}", csr, sc, ctx, cfg))
    return cases


def arrays_digest(csr) -> str:
    h = hashlib.sha256()
    for a, dt in ((csr.row_offsets, np.int64), (csr.ilabels, np.int64), (csr.olabels, np.int64),
                  (csr.next_states, np.int64), (csr.weights, np.float64)):
        h.update(np.ascontiguousarray(a, dtype=dt).tobytes())
    return h.hexdigest()


def c1_small() -> tuple[dict, dict]:
    t0 = time.time()
    fst = build_benchmark_graph(10_000, 4, 2000, eps_input_frac=0.1, seed=421)
    csr = build_csr(fst)
    digest = {"g_small": arrays_digest(csr), "fingerprint": csr.fingerprint,
              "num_arcs": int(csr.num_arcs)}
    words = random.Random(1).sample(range(1, 2001), 20)
    idx = np.flatnonzero(np.isin(csr.olabels, words)).astype(np.int64)
    ctx = BiasingContext(id="ctx1", arc_indices=idx, discount=-2.0)
    cfg = DecoderConfig(beam=13.0, max_active=7000, max_epsilon_expansion=20, partial_every=10)
    out = {"graph": "benchmark_graph(10000, 4, 2000, seed=421)", "ctx_words": words,
           "ctx_arcs": [int(v) for v in idx], "cfg": cfg_json(cfg), "runs": {}}
    T = 500
    scores = np.random.default_rng([7, 0]).uniform(0.0, 6.0, (T, 2000))
    out["runs"]["f64"] = run_ref(csr, scores, ctx, cfg)
    # f32 variant: weights and scores rounded once to float32
    w32 = csr.weights.astype(np.float32).astype(np.float64)
    csr32 = CsrFst(start=csr.start, row_offsets=csr.row_offsets, ilabels=csr.ilabels,
                   olabels=csr.olabels, next_states=csr.next_states, weights=w32,
                   finals=csr.finals, fingerprint="")
    s32 = scores.astype(np.float32).astype(np.float64)
    out["runs"]["f32"] = run_ref(csr32, s32, ctx, cfg)
    out["runs"]["f32_unbiased"] = run_ref(csr32, s32, None, cfg)
    print(f"c1 reference runs: {time.time() - t0:.1f}s")
    return out, digest


def margin_suite() -> dict:
    suite = build_margin_suite(50)
    csr = build_csr(suite.fst)
    ctx = compile_context(suite.fst, suite.symtab, suite.entities, BoostCompileConfig(), id="ents")
    cfg = DecoderConfig()
    utts = []
    for u in suite.utterances:
        utts.append({
            "utt_id": u.utt_id,
            "scores": [[hx(v) for v in row] for row in u.scores.costs],
            "transcript": [suite.symtab.id_of(w) for w in u.transcript],
            "unbiased": run_ref(csr, u.scores.costs, None, cfg),
            "biased": run_ref(csr, u.scores.costs, ctx, cfg),
        })
    return {"graph": graph_json(csr), "ctx": {"arc_indices": [int(v) for v in ctx.arc_indices],
                                              "discount": hx(ctx.discount)},
            "cfg": cfg_json(cfg), "utts": utts}


def main() -> None:
    (OUT / "small_cases.json").write_text(json.dumps(small_cases()))
    c1, digest = c1_small()
    (OUT / "c1_small.json").write_text(json.dumps(c1))
    (OUT / "graph_digest.json").write_text(json.dumps(digest, indent=1))
    (OUT / "margin_suite.json").write_text(json.dumps(margin_suite()))
    print("written:", sorted(p.name for p in OUT.glob("*.json")))


if __name__ == "__main__":
    main()
