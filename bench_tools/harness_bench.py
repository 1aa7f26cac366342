"""Run-harness benchmark: a whole ``run_decode`` — score
files parsed, contexts compiled from entity files, waves decoded, WER scored,
JSONL written — on the same generated inputs through this package (GPU) or
the reference package (CPU, this container only).

    python bench_tools/harness_bench.py --make /tmp/hb            # write inputs
    python bench_tools/harness_bench.py --dir /tmp/hb --impl ours
    python bench_tools/harness_bench.py --dir /tmp/hb --impl reference

Inputs (deterministic): G_small (benchmark_graph(10_000, 4, 2000), f32
weights) as a text graph, a 2000-word symbol table, 8 entity files of 20
single words, C channels x U utterances x T frames of U[0, 6) costs as score
files, references of 10 random words with 2 entity words.  One JSON line:
timings, RTFX, WER, and SHA-256 of the report (clocks removed) and of the
JSONL stream, so two machines' outputs can be compared.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import random
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def make(d: Path, channels: int, utts: int, frames: int) -> None:
    from paper_2306_15685_b200 import synth

    d.mkdir(parents=True, exist_ok=True)
    csr = synth.benchmark_graph(10_000, 4, 2000, seed=421, f32_weights=True)
    ro, il, ol, ns, w = (np.asarray(a) for a in (csr.row_offsets, csr.ilabels, csr.olabels,
                                                  csr.next_states, csr.weights))
    lines = []
    for s in range(len(ro) - 1):
        for a in range(ro[s], ro[s + 1]):
            lines.append(f"{s} {ns[a]} {il[a]} {ol[a]} {float(w[a])!r}")
    lines += [f"{s} 0.0" for s in range(len(ro) - 1)]
    (d / "graph.fst").write_text("\n".join(lines) + "\n")
    (d / "words.txt").write_text("<eps> 0\n" + "".join(f"w{i} {i}\n" for i in range(1, 2001)))
    rng = random.Random(7)
    ctx_words = []
    for k in range(8):
        ws = rng.sample(range(1, 2001), 20)
        ctx_words.append(ws)
        (d / f"ctx{k}.txt").write_text("".join(f"w{x}\n" for x in ws))
    (d / "contexts.tsv").write_text("".join(f"ctx{k}\t{d}/ctx{k}.txt\n" for k in range(8)))
    rows = []
    for c in range(channels):
        for u in range(utts):
            uid = f"c{c}u{u}"
            x = np.random.default_rng([11, c, u]).uniform(0.0, 6.0, (frames, 2000))
            x = x.astype(np.float32).astype(np.float64)
            body = "\n".join(" ".join(repr(v) for v in row) for row in x.tolist())
            (d / f"{uid}.scores").write_text(f"{frames} 2000 0.03\n{body}\n")
            k = (c + u) % 8
            ents = rng.sample(ctx_words[k], 2)
            ref = [f"w{rng.randint(1, 2000)}" for _ in range(8)] + [f"w{e}" for e in ents]
            rng.shuffle(ref)
            rows.append(f"{uid}\tch{c}\t{d}/{uid}.scores\tctx{k}\t{' '.join(ref)}\t"
                        f"{'|'.join(f'w{e}' for e in ents)}\n")
    (d / "utts.tsv").write_text("".join(rows))


def run(d: Path, impl: str, repeats: int) -> dict:
    t0 = time.perf_counter()
    if impl == "reference":
        sys.path.insert(0, "/root/reference/pkg/src")
        sys.dont_write_bytecode = True
        from arcboost.biasing import BoostCompileConfig, load_registry, read_context_manifest
        from arcboost.decoder import DecoderConfig
        from arcboost.fst import build_csr, parse_symbol_table, parse_text_fst
        from arcboost.harness import read_utterance_specs, run_decode

        fst = parse_text_fst((d / "graph.fst").read_text())
        csr = build_csr(fst)
        graph = fst
    else:
        from paper_2306_15685_b200 import (BoostCompileConfig, DecoderConfig, load_registry,
                                           parse_symbol_table, read_context_manifest)
        from paper_2306_15685_b200.fst import parse_text_fst_csr
        from paper_2306_15685_b200.harness import read_utterance_specs, run_decode

        csr = parse_text_fst_csr((d / "graph.fst").read_bytes())
        graph = csr
    symtab = parse_symbol_table((d / "words.txt").read_text())
    t_graph = time.perf_counter() - t0
    t1 = time.perf_counter()
    registry = load_registry(graph, symtab, read_context_manifest((d / "contexts.tsv").read_text()),
                             BoostCompileConfig())
    t_ctx = time.perf_counter() - t1
    specs = read_utterance_specs((d / "utts.tsv").read_text())
    cfg = DecoderConfig(beam=13.0, max_active=7000, partial_every=10)
    runs = []
    for _ in range(repeats):
        report, jsonl = run_decode(csr, symtab, registry, specs, cfg)
        runs.append(report.timing | {"rtfx": report.rtfx})
    rep = json.loads(report.to_json())
    del rep["timing"], rep["rtfx"]
    frames = sum(int(open(s.score_path).readline().split()[0]) for s in specs)
    return {"impl": impl, "utterances": len(specs), "frames": frames, "graph_s": t_graph,
            "contexts_s": t_ctx, "runs": runs, "wer": report.wer, "ent_wer": report.ent_wer,
            "report_sha256": hashlib.sha256(json.dumps(rep, sort_keys=True).encode()).hexdigest(),
            "jsonl_sha256": hashlib.sha256("\n".join(jsonl).encode()).hexdigest(),
            "jsonl_lines": len(jsonl)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--make", type=Path)
    ap.add_argument("--dir", type=Path)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--channels", type=int, default=32)
    ap.add_argument("--utts", type=int, default=2)
    ap.add_argument("--frames", type=int, default=50)
    ap.add_argument("--repeats", type=int, default=2)
    a = ap.parse_args()
    if a.make:
        make(a.make, a.channels, a.utts, a.frames)
        return
    print(json.dumps(run(a.dir, a.impl, a.repeats)))


if __name__ == "__main__":
    main()
