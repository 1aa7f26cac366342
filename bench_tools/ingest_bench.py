"""Graph ingest: text FST -> CSR + reference fingerprint.
Native (ab_fst_load) on the C3 graph's text (5M states / 20M arcs) cold and
from the binary cache; the reference's parse_text_fst + build_csr +
fingerprint on a smaller graph (Python does not scale to 20M arcs).  CPU
only; prints one JSON line.  The reference part runs only where
/root/reference exists."""
import json
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2306_15685_b200 import fst as M, synth  # noqa: E402


def write_text(csr, path):
    S = csr.num_states
    src = np.repeat(np.arange(S, dtype=np.int64), np.diff(csr.row_offsets))
    with open(path, "w") as f:
        # start state's lines first (the first line names the start)
        order = np.argsort(src != csr.start, kind="stable")
        cols = np.stack([src[order], csr.next_states[order], csr.ilabels[order], csr.olabels[order]], 1)
        w = csr.weights[order]
        chunk = 1 << 20
        for i in range(0, len(cols), chunk):
            f.write("".join(f"{a} {b} {c} {d} {x!r}\n" for (a, b, c, d), x in
                            zip(cols[i:i + chunk].tolist(), w[i:i + chunk].tolist())))
        for s, c in sorted(csr.finals.items()):
            f.write(f"{s} {c!r}\n")


def main():
    res = {"what": "text FST -> state-major CSR + reference fingerprint"}
    tmp = Path(tempfile.mkdtemp())
    big = synth.benchmark_graph(int(os.environ.get("INGEST_STATES", 5_000_000)), 4, 2000, seed=421,
                                f32_weights=True)
    p = tmp / "g_large.txt"
    write_text(big, p)
    t0 = time.perf_counter()
    a = M.load_fst(p, cache=True)
    t1 = time.perf_counter()
    b = M.load_fst(p, cache=True)
    t2 = time.perf_counter()
    res["native"] = {"states": a.num_states, "arcs": a.num_arcs, "text_MB": p.stat().st_size / 1e6,
                     "parse_s": t1 - t0, "cache_load_s": t2 - t1, "cache_hit": b.cache_hit,
                     "arrays_equal_generator": bool(np.array_equal(a.next_states, big.next_states))}
    ref = Path("/root/reference/pkg/src")
    if ref.exists():
        sys.path.insert(0, str(ref))
        sys.dont_write_bytecode = True
        from arcboost.fst import build_csr, parse_text_fst
        small = synth.benchmark_graph(100_000, 4, 2000, seed=421, f32_weights=True)
        q = tmp / "g_small.txt"
        write_text(small, q)
        t0 = time.perf_counter()
        r = build_csr(parse_text_fst(q.read_text()))
        fp = r.fingerprint
        t1 = time.perf_counter()
        n = M.load_fst(q, cache=False)
        t2 = time.perf_counter()
        res["reference_python"] = {"states": 100_000, "arcs": int(r.row_offsets[-1]), "seconds": t1 - t0}
        res["native_same_graph"] = {"seconds": t2 - t1, "fingerprint_equal": n.fingerprint == fp,
                                    "arrays_equal": bool(np.array_equal(n.next_states, r.next_states))
                                    and bool(np.array_equal(n.weights, r.weights))}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
