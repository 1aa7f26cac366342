import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2306_15685_b200 as ab
from paper_2306_15685_b200 import synth, _lib
from oracle.oracle import OracleChannel, OracleGraph
csr = synth.benchmark_graph(10_000, 4, 2000, seed=421, f32_weights=True)
ctx = synth.unigram_context(csr, 20, 3, num_labels=2000)
og = OracleGraph.from_csr(csr)
for exact in (True, False):
    cfg = ab.DecoderConfig(beam=13.0, max_active=3000, exact_counters=exact)
    och = OracleChannel(og)
    ch = ab.init_channel("t", None, None, cfg)
    scores = synth.channel_scores(5, 0, 12, 2000)
    for t in range(12):
        ab.advance_frame(ch, scores[t], csr, ctx, cfg)
        och.advance(scores[t].astype(np.float64), ctx, cfg)
        st, co, hi = och.tokens()
        toks = ch.active_tokens()
        ok = [x.state for x in toks] == st.tolist() and [x.cost for x in toks] == co.tolist()
        info = ch._page.get(ch._slot)
        ds = [x.state for x in toks]
        dup = len(ds) - len(set(ds))
        extra = sorted(set(ds) - set(st.tolist()))[:5]
        missing = sorted(set(st.tolist()) - set(ds))[:5]
        if not ([x.state for x in toks] == st.tolist()):
            print("  dup", dup, "extra", extra, "missing", missing, "max dev cost", max(x.cost for x in toks), "max orc cost", co.max(), "min", min(x.cost for x in toks), co.min())
        print(os.environ.get("AB_CLUSTER"), "exact", exact, "frame", t, "dev", len(toks), "orc", len(st), "ok", ok, "redos", info.cut_redos, "store", len(ch.store), och.info()["store_len"])
        if not ok:
            break
