"""Dense-context (C4 5%) cutoff cost: slack, flagged states, per-segment kernel
time and expanded work, unbiased vs zero-discount vs -2.0 contexts."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2306_15685_b200 as ab  # noqa: E402
from paper_2306_15685_b200 import _lib, synth  # noqa: E402
from paper_2306_15685_b200.device import BatchDecoder, Capacity, DeviceGraph  # noqa: E402

L = 2000
csr = synth.benchmark_graph(5_000_000, 4, L, seed=421, f32_weights=True)
dg = DeviceGraph(csr, 0)
C, T = 256, 125
dec = BatchDecoder(dg, C, Capacity(arena_records=1 << 20))
scores = synth.device_channel_scores(7, range(C), T, L, device=0)
import torch  # noqa: E402
torch.cuda.synchronize()
cfg = ab.DecoderConfig(beam=13.0, max_active=7000, max_epsilon_expansion=20, partial_every=10)
slots = np.arange(C, dtype=np.int32)
for kind in ("words", "arcs"):
    for dens in (0.01, 0.05):
        if kind == "words":
            pool = synth.unigram_contexts(csr, int(dens * L), range(2000, 2004), num_labels=L)
        else:
            pool = [synth.dense_context(csr, dens, 2000 + i) for i in range(4)]
        variants = {"unbiased": [-1] * 4,
                    "zero": [dg.register_context(c.arc_indices, 0.0) for c in pool],
                    "-2": [dg.register_context(c.arc_indices, -2.0) for c in pool]}
        print(kind, dens, "slack/flagged -2:", [tuple(round(x, 2) for x in dg.context_slack(h)) for h in variants["-2"]])
        for name, hs in variants.items():
            for rep in range(2):
                dec.init_channels(slots, [hs[c % 4] for c in range(C)])
                dec.decode(slots, np.full(C, T, np.int32), np.arange(C, dtype=np.int64) * T * L, scores.data_ptr(),
                           L, cfg, _lib.AB_MODE_STREAM, scores_on_device=True, scores_dtype=_lib.AB_F32)
                nh, er, *_ = dec.results(C)
                inf = dec.get_many(slots)
            n = np.mean([i.tok_expansions for i in inf]) / T
            ax = np.mean([i.eps_arcs for i in inf]) / T
            print(f"  {name:9s} kernel {dec.last_kernel_ms():7.1f} ms  N/cf {n:7.0f}  A_eps/cf {ax:6.0f}  "
                  f"redos {sum(i.cut_redos for i in inf)} err {int((er != 0).sum())}")
        for h in variants["zero"] + variants["-2"]:
            dg.release_context(h)
