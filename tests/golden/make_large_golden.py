"""G_large golden fixture: the REFERENCE decoder (read-only import from
/root/reference/pkg/src) run on the C3 benchmark graph, in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_large_golden.py

Graph: the arrays of ``synth.benchmark_graph(5_000_000, 4, 2000, seed=421,
f32_weights=True)`` (the draws of the reference's build_benchmark_graph,
synth.py:294-322, vectorised; weights rounded once to f32) wrapped in the
reference's own ``CsrFst`` with every state final at 0.0 (synth.py:321) -
the reference decodes G_large through ``CsrFst``.

Runs (all with beam 13, max_active 7000, max_epsilon_expansion 20,
partial_every 10; reference harness waves, harness.py:208-242: every segment
is one utterance, ``switch_context`` between segments on the same Channel):

  c3       bench.py's C3 channels 0..3, segments 0 and 1 (125 frames each),
           contexts from the bench pool (256 twenty-word unigram contexts,
           ctx_index(c, seg)), scores default_rng([7, c]) U[0,6) as f32 -
           exactly the first two segments the GPU bench decodes for them;
           plus channel 4 unbiased in segment 0 and biased in segment 1
  c4       60 frames of one channel with a 100-word context (~5% of arcs,
           label-closed) and one with 5% of arcs drawn uniformly (not
           label-closed: the BITSET representation on the device)

Only inputs' recipes and outputs are stored (hypotheses bit-exact as
float.hex, len(store), eps_truncations, utterance_index), plus a digest of
the graph arrays so the GPU test knows it rebuilt the same graph.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from arcboost.biasing import BiasingContext, ContextRegistry  # noqa: E402
from arcboost.decoder import DecoderConfig, decode_batch, init_channel, switch_context  # noqa: E402
from arcboost.fst import CsrFst  # noqa: E402
from arcboost.scores import ScoreMatrix  # noqa: E402

from paper_2306_15685_b200 import synth  # noqa: E402  (input generator only)

OUT = Path(__file__).resolve().parent / "g_large.json"
L = 2000
POOL = 256
SEG = 125


def hx(x: float) -> str:
    return float(x).hex()


def ctx_index(c: int, seg: int, n_pool: int) -> int:  # bench.py
    return (c * 131 + seg * 17) % n_pool


def digest(csr) -> str:
    h = hashlib.sha256()
    for a, dt in ((csr.row_offsets, np.int64), (csr.ilabels, np.int64), (csr.olabels, np.int64),
                  (csr.next_states, np.int64), (csr.weights, np.float64)):
        h.update(np.ascontiguousarray(a, dtype=dt).tobytes())
    return h.hexdigest()


def hyps_json(res) -> dict:
    return {"error": res.error,
            "hyps": [{"words": h.words, "cost": hx(h.cost), "frame": h.frame, "kind": h.kind,
                      "fallback": h.fallback} for h in res.hypotheses]}


def main() -> None:
    t0 = time.time()
    g = synth.benchmark_graph(5_000_000, 4, L, seed=421, f32_weights=True)
    n_states = len(g.row_offsets) - 1
    csr = CsrFst(start=0, row_offsets=np.asarray(g.row_offsets, dtype=np.int64),
                 ilabels=np.asarray(g.ilabels, dtype=np.int64),
                 olabels=np.asarray(g.olabels, dtype=np.int64),
                 next_states=np.asarray(g.next_states, dtype=np.int64),
                 weights=np.asarray(g.weights, dtype=np.float64),
                 finals={s: 0.0 for s in range(n_states)}, fingerprint="")
    pool = synth.unigram_contexts(g, 20, range(1000, 1000 + POOL), num_labels=L)
    ref_pool = {c.id: BiasingContext(id=c.id, arc_indices=np.asarray(c.arc_indices, dtype=np.int64),
                                     discount=c.discount) for c in pool}
    reg = ContextRegistry(contexts=ref_pool, graph_fingerprint="")
    cfg = DecoderConfig(beam=13.0, max_active=7000, max_epsilon_expansion=20, partial_every=10)
    print(f"graph + contexts: {time.time() - t0:.1f}s", flush=True)

    chans = list(range(5))
    plan = {c: [pool[ctx_index(c, s, POOL)].id for s in range(2)] for c in range(4)}
    plan[4] = [None, pool[ctx_index(4, 1, POOL)].id]
    mats = {c: synth.channel_scores(7, c, 2 * SEG, L).astype(np.float64) for c in chans}
    ref_ch = {c: init_channel(f"c{c}", reg, None, cfg) for c in chans}
    out = {"graph": "benchmark_graph(5_000_000, 4, 2000, seed=421, f32_weights=True)",
           "digest": digest(g), "cfg": {"beam": 13.0, "max_active": 7000,
                                        "max_epsilon_expansion": 20, "partial_every": 10},
           "pool": {"num_words": 20, "seeds": [1000, 1000 + POOL]}, "seg_frames": SEG,
           "scores": "synth.channel_scores(7, c, 250, 2000) (f32), segment s = rows [125 s, 125 s + 125)",
           "c3": []}
    for seg in range(2):
        t1 = time.time()
        batch = []
        for c in chans:
            switch_context(ref_ch[c], reg, plan[c][seg])
            batch.append((ref_ch[c], ScoreMatrix(costs=mats[c][seg * SEG:(seg + 1) * SEG])))
        res = decode_batch(batch, csr, reg, cfg)
        for c, r in zip(chans, res):
            ch = ref_ch[c]
            out["c3"].append({"channel": c, "segment": seg, "context": plan[c][seg], **hyps_json(r),
                              "store_len": len(ch.store), "eps_truncations": ch.eps_truncations,
                              "utterance_index": ch.utterance_index})
        print(f"segment {seg}: {time.time() - t1:.1f}s", flush=True)

    # C4: dense contexts (60 frames of channel 0's scores)
    words100 = synth.unigram_contexts(g, 100, [2000], num_labels=L)[0]
    dense = synth.dense_context(g, 0.05, 2000)
    out["c4"] = []
    for name, ctx in (("words100", words100), ("arcs5pct", dense)):
        t1 = time.time()
        rc = BiasingContext(id=name, arc_indices=np.asarray(ctx.arc_indices, dtype=np.int64),
                            discount=-2.0)
        r4 = ContextRegistry(contexts={name: rc}, graph_fingerprint="")
        ch = init_channel(name, r4, name, cfg)
        res = decode_batch([(ch, ScoreMatrix(costs=mats[0][:60]))], csr, r4, cfg)[0]
        out["c4"].append({"name": name, "k": int(len(rc.arc_indices)), **hyps_json(res),
                          "store_len": len(ch.store), "eps_truncations": ch.eps_truncations})
        print(f"c4 {name}: {time.time() - t1:.1f}s", flush=True)
    out["c4_recipe"] = {"words100": "synth.unigram_contexts(g, 100, [2000], num_labels=2000)[0]",
                        "arcs5pct": "synth.dense_context(g, 0.05, 2000)", "discount": -2.0,
                        "scores": "channel 0, rows [0, 60)"}
    OUT.write_text(json.dumps(out))
    print(f"written {OUT} in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
