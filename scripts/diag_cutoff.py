"""Cutoff diagnostics on the C3 workload: per-context epsilon slack and flagged
states, and per-channel work (expanded token / epsilon-arc counts, redone
frames) for one biased and one unbiased 125-frame segment of 256 channels."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2306_15685_b200 as ab  # noqa: E402
from paper_2306_15685_b200 import _lib, synth  # noqa: E402
from paper_2306_15685_b200.device import BatchDecoder, Capacity, DeviceGraph  # noqa: E402

L = 2000
csr = synth.benchmark_graph(5_000_000, 4, L, seed=421, f32_weights=True)
pool = synth.unigram_contexts(csr, 20, range(1000, 1256), num_labels=L)
dg = DeviceGraph(csr, 0)
hs = [dg.register_context(c.arc_indices, c.discount) for c in pool]
sl = np.array([dg.context_slack(h) for h in hs])
print("graph slack", dg.context_slack(-1))
print("slack: min %.3f median %.3f max %.3f  inf %d; flagged bits median %d max %d" % (
    sl[:, 0].min(), np.median(sl[:, 0]), sl[np.isfinite(sl[:, 0]), 0].max(), np.isinf(sl[:, 0]).sum(),
    np.median(sl[:, 1]), sl[:, 1].max()))
C, T = 256, 125
dec = BatchDecoder(dg, C, Capacity(arena_records=1 << 20))
scores = synth.device_channel_scores(7, range(C), T, L, device=0)
import torch  # noqa: E402
torch.cuda.synchronize()
cfg = ab.DecoderConfig(beam=13.0, max_active=7000, max_epsilon_expansion=20, partial_every=10)
slots = np.arange(C, dtype=np.int32)
for name, ctx in [("unbiased", [-1] * C), ("biased", [hs[(c * 131) % 256] for c in range(C)])]:
    for exact in (False, True):
        c2 = ab.DecoderConfig(beam=13.0, max_active=7000, max_epsilon_expansion=20, partial_every=10,
                              exact_counters=exact)
        dec.init_channels(slots, ctx)
        t0 = time.time()
        dec.decode(slots, np.full(C, T, np.int32), np.arange(C, dtype=np.int64) * T * L, scores.data_ptr(), L,
                   c2, _lib.AB_MODE_STREAM, scores_on_device=True, scores_dtype=_lib.AB_F32)
        nh, er, *_ = dec.results(C)
        ms = dec.last_kernel_ms()
        inf = dec.get_many(slots)
        n = np.array([i.tok_expansions for i in inf]) / T
        ax = np.array([i.eps_arcs for i in inf]) / T
        rd = np.array([i.cut_redos for i in inf])
        print(f"{name:9s} exact={exact}: kernel {ms:.1f} ms; N/cf median {np.median(n):.0f} p10 {np.percentile(n, 10):.0f} "
              f"p90 {np.percentile(n, 90):.0f}; A_eps/cf median {np.median(ax):.0f}; redos total {rd.sum()} "
              f"max/ch {rd.max()}; errors {int((er != 0).sum())}")
        if name == "biased" and not exact:
            worst = np.argsort(-n)[:5]
            print("  heaviest channels", worst.tolist(), n[worst].round(0).tolist(), "slack",
                  [sl[(c * 131) % 256].tolist() for c in worst])
