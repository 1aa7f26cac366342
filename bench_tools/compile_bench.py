"""Alg. 1 context compilation at scale: the native compiler
(ab_compile_context, all host threads) on G_large, and the reference's Python
find_boost_arcs on a mid-size graph it can hold (its adjacency-list Fst and the
all-arcs scan per first word do not scale to 20M arcs).  CPU only; prints one
JSON line.  The reference part runs only where /root/reference exists.

    python bench_tools/compile_bench.py [--states 5000000] [--entities 5120]
"""
import argparse
import json
import os
import random
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2306_15685_b200 import compiler as K, synth  # noqa: E402


def entities(csr, n, seed):
    """Multi-word entities that exist in the graph: random 2-3 arc walks that
    output a word at each step (so Alg. 1 has chains to follow)."""
    import numpy as np
    rng = random.Random(seed)
    ro, ol, ns = csr.row_offsets, csr.olabels, csr.next_states
    out = []
    while len(out) < n:
        g = rng.randrange(len(ol))
        words = []
        for _ in range(rng.randint(2, 3)):
            if ol[g] == 0:
                break
            words.append(int(ol[g]))
            s = int(ns[g])
            if ro[s + 1] == ro[s]:
                break
            g = rng.randrange(int(ro[s]), int(ro[s + 1]))
        if len(words) >= 2:
            out.append(words)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--states", type=int, default=5_000_000)
    ap.add_argument("--entities", type=int, default=5120)  # 256 contexts x 20 entities
    ap.add_argument("--ref-states", type=int, default=20_000)
    ap.add_argument("--ref-entities", type=int, default=40)
    a = ap.parse_args()
    res = {"what": "Alg. 1 context compilation (find_boost_arcs over multi-word entities)"}
    csr = synth.benchmark_graph(a.states, 4, 2000, seed=421, f32_weights=True)
    ents = entities(csr, a.entities, 1)
    arrays = K.csr_arrays(csr)
    t0 = time.perf_counter()
    arcs, status = K._compile(arrays, ents, 10, os.cpu_count() or 1)
    dt = time.perf_counter() - t0
    res["native"] = {"graph_states": a.states, "graph_arcs": int(csr.row_offsets[-1]),
                     "entities": len(ents), "seconds": dt, "entities_per_s": len(ents) / dt,
                     "threads": os.cpu_count(), "boosted_arcs": int(len(arcs)),
                     "compiled": int((status == 1).sum())}
    ref = Path("/root/reference/pkg/src")
    if ref.exists():
        sys.path.insert(0, str(ref))
        sys.dont_write_bytecode = True
        from arcboost.biasing import BoostCompileConfig, find_boost_arcs
        from arcboost.synth import build_benchmark_graph
        fst = build_benchmark_graph(num_states=a.ref_states, arcs_per_state=4, num_labels=2000,
                                    eps_input_frac=0.1, seed=421)
        small = synth.benchmark_graph(a.ref_states, 4, 2000, seed=421)
        ents_s = entities(small, a.ref_entities, 2)
        t0 = time.perf_counter()
        want = sorted({g for e in ents_s for g in find_boost_arcs(fst, e, BoostCompileConfig())})
        dt_ref = time.perf_counter() - t0
        t0 = time.perf_counter()
        got, _ = K._compile(K.csr_arrays(small), ents_s, 10, 1)
        dt_nat = time.perf_counter() - t0
        res["reference_python"] = {"graph_states": a.ref_states, "entities": len(ents_s),
                                   "seconds": dt_ref, "entities_per_s": len(ents_s) / dt_ref}
        res["native_same_sample_1_thread"] = {"seconds": dt_nat, "entities_per_s": len(ents_s) / dt_nat,
                                              "identical_to_reference": got.tolist() == want}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
