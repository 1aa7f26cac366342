import cProfile, pstats, sys, time
sys.path.insert(0, '.')
from pathlib import Path
from paper_2306_15685_b200 import BoostCompileConfig, DecoderConfig, load_registry, parse_symbol_table, read_context_manifest
from paper_2306_15685_b200.fst import parse_text_fst_csr
from paper_2306_15685_b200.harness import read_utterance_specs, run_decode
d = Path(sys.argv[1])
csr = parse_text_fst_csr((d / "graph.fst").read_bytes())
st = parse_symbol_table((d / "words.txt").read_text())
reg = load_registry(csr, st, read_context_manifest((d / "contexts.tsv").read_text()), BoostCompileConfig())
specs = read_utterance_specs((d / "utts.tsv").read_text())
cfg = DecoderConfig(beam=13.0, max_active=7000, partial_every=10)
run_decode(csr, st, reg, specs, cfg)
pr = cProfile.Profile(); pr.enable()
r, _ = run_decode(csr, st, reg, specs, cfg)
pr.disable()
print(r.timing)
pstats.Stats(pr).sort_stats('cumulative').print_stats(30)
