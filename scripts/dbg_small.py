"""Decodes the reference small cases one by one (tests/ inputs) and reports
the first one that errors or differs; for compute-sanitizer runs.
argv[1] = 'exact' | 'cutoff', argv[2] = max cases."""
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)
import conftest as T  # noqa: E402
from test_gpu_parity import _decode  # noqa: E402

exact = len(sys.argv) > 1 and sys.argv[1] == "exact"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
for c in T.load_json("small_cases.json")[:n]:
    csr, scores, ctx, cfg = T.case_inputs(c, exact)
    try:
        res, ch = _decode(csr, scores, ctx, cfg)
    except Exception as e:  # a CUDA fault ends the process's context: report and stop
        print("FAIL", c["name"], repr(e)[:300], flush=True)
        sys.exit(1)
    e = c["expect"]
    got = [(h.words, h.cost, h.frame, h.kind, h.fallback) for h in res.hypotheses]
    ok = (res.error is not None) if e["error"] is not None else (res.error is None and got == T.expect_hyps(e))
    print("ok" if ok else "DIFF", c["name"], flush=True)
