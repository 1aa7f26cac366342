"""LIST-context cost on C3: kernel time and work counters of one 125-frame
segment of 256 channels, unbiased vs zero-discount entity contexts (LIST hash
set) vs the same arc sets as BITSET, vs -2.0 discount."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2306_15685_b200 as ab  # noqa: E402
from paper_2306_15685_b200 import _lib, synth  # noqa: E402
from paper_2306_15685_b200.device import BatchDecoder, Capacity, DeviceGraph  # noqa: E402

L = 2000
csr = synth.benchmark_graph(5_000_000, 4, L, seed=421, f32_weights=True)
pool = synth.entity_contexts(csr, 20, range(1000, 1032))
dg = DeviceGraph(csr, 0)
C, T = 256, 125
dec = BatchDecoder(dg, C, Capacity(arena_records=1 << 20))
scores = synth.device_channel_scores(7, range(C), T, L, device=0)
import torch  # noqa: E402
torch.cuda.synchronize()
cfg = ab.DecoderConfig(beam=13.0, max_active=7000, max_epsilon_expansion=20, partial_every=10)
slots = np.arange(C, dtype=np.int32)
variants = {
    "unbiased": [-1] * len(pool),
    "zero LIST": [dg.register_context(c.arc_indices, 0.0) for c in pool],
    "zero BITSET": [dg.register_context(c.arc_indices, 0.0, _lib.AB_CTX_BITSET) for c in pool],
    "-2 LIST": [dg.register_context(c.arc_indices, -2.0) for c in pool],
    "-2 BITSET": [dg.register_context(c.arc_indices, -2.0, _lib.AB_CTX_BITSET) for c in pool],
}
print("modes", {k: (dg.context_mode(v[0]) if v[0] >= 0 else None) for k, v in variants.items()})
print("slack -2", [dg.context_slack(h) for h in variants["-2 LIST"][:4]])
for name, hs in variants.items():
    for rep in range(2):
        dec.init_channels(slots, [hs[c % len(hs)] for c in range(C)])
        dec.decode(slots, np.full(C, T, np.int32), np.arange(C, dtype=np.int64) * T * L, scores.data_ptr(), L,
                   cfg, _lib.AB_MODE_STREAM, scores_on_device=True, scores_dtype=_lib.AB_F32)
        nh, er, *_ = dec.results(C)
        inf = dec.get_many(slots)
    n = np.mean([i.tok_expansions for i in inf]) / T
    ax = np.mean([i.eps_arcs for i in inf]) / T
    print(f"{name:12s} kernel {dec.last_kernel_ms():7.1f} ms  N/cf {n:7.0f}  A_eps/cf {ax:6.0f}  redos {sum(i.cut_redos for i in inf)} err {int((er != 0).sum())}")
