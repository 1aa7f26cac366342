"""Run harness and scoring against the reference:
tests/golden/harness_cases.json (tests/golden/make_harness_golden.py runs the
reference's metrics, symbol-table / manifest readers and whole run_decode
calls).  Scoring and readers are CPU tests; run_decode parity is a GPU test
(the decode runs on the device) and compares the report and the JSONL
hypothesis stream byte for byte."""

import json

import pytest

from conftest import F1_TEXT, load_json

import paper_2306_15685_b200 as ab
from paper_2306_15685_b200 import harness as H
from paper_2306_15685_b200 import metrics as M
from paper_2306_15685_b200.fst import parse_text_fst_csr


@pytest.fixture(scope="module")
def golden():
    return load_json("harness_cases.json")


def raises_like(e: dict, fn, *args):
    with pytest.raises(Exception) as ei:
        fn(*args)
    assert type(ei.value).__name__ == e["type"]
    assert str(ei.value) == e["message"]


# ------------------------------------------------------------------ scoring

def test_align_matches_reference(golden):
    for i, c in enumerate(golden["align"]):
        ops = M.align(c["ref"], c["hyp"])
        assert [[o.kind, o.ref_pos, o.hyp_pos] for o in ops] == c["ops"], i
        assert list(M.edit_counts(ops)) == c["counts"], i


def test_wer_matches_reference(golden):
    for i, c in enumerate(golden["wer"]):
        pairs = [tuple(p) for p in c["pairs"]]
        if "error" in c:
            raises_like(c["error"], M.compute_wer, pairs)
        else:
            assert M.compute_wer(pairs) == c["wer"], i


def test_ent_wer_matches_reference(golden):
    for i, c in enumerate(golden["ent_wer"]):
        for ref, ents, spans in zip(c["refs"], c["entities"], c["spans"]):
            assert [list(s) for s in M.locate_entity_spans(ref, ents)] == spans, i
        if "error" in c:
            raises_like(c["error"], M.compute_ent_wer, c["refs"], c["hyps"], c["entities"])
        else:
            assert M.compute_ent_wer(c["refs"], c["hyps"], c["entities"]) == c["ent_wer"], i


def test_reference_metric_examples():
    # reference tests/test_metrics.py: kinds of simple alignments, RTFX
    assert [o.kind for o in M.align(["a", "b", "c"], ["a", "x", "c"])] == [M.MATCH, M.SUBSTITUTION, M.MATCH]
    assert [o.kind for o in M.align([], ["a"])] == [M.INSERTION]
    assert sum(M.edit_counts(M.align(["a", "b"], ["a", "b"]))) == 0
    assert M.compute_rtfx(10.0, 2.0) == 5.0
    with pytest.raises(M.ScoringError):
        M.compute_rtfx(1.0, 0.0)
    with pytest.raises(M.ScoringError):
        M.compute_wer([([], ["a"])])


def test_edit_distances_batch_threads():
    import random
    rng = random.Random(5)
    pairs = [([rng.choice("abc") for _ in range(rng.randint(0, 40))],
              [rng.choice("abc") for _ in range(rng.randint(0, 40))]) for _ in range(300)]
    one = M.edit_distances(pairs, threads=1)
    many = M.edit_distances(pairs, threads=8)
    assert one.tolist() == many.tolist()
    assert one.tolist() == [sum(M.edit_counts(M.align(r, h))) for r, h in pairs]


# ------------------------------------------------------------------ readers

def test_symbol_tables_match_reference(golden):
    for c in golden["symtabs"]:
        if "error" in c:
            raises_like(c["error"], ab.parse_symbol_table, c["text"])
        else:
            st = ab.parse_symbol_table(c["text"])
            assert {w: st.id_of(w) for w in st.words()} == c["words"]
            for w, i in c["words"].items():
                assert st.word_of(i) == w


def test_manifests_match_reference(golden):
    import dataclasses
    m = golden["manifests"]
    for c in m["utterances"]:
        if "error" in c:
            raises_like(c["error"], H.read_utterance_specs, c["text"])
        else:
            specs = H.read_utterance_specs(c["text"])
            assert [dataclasses.asdict(s) for s in specs] == c["rows"]
            assert H.read_utterance_specs(H.format_utterance_specs(specs)) == specs
    for c in m["transcripts"]:
        if "error" in c:
            raises_like(c["error"], H.read_transcripts, c["text"])
        else:
            assert [dataclasses.asdict(s) for s in H.read_transcripts(c["text"])] == c["rows"]
    for c in m["contexts"]:
        if "error" in c:
            raises_like(c["error"], ab.read_context_manifest, c["text"])
        else:
            assert [list(r) for r in ab.read_context_manifest(c["text"])] == c["rows"]


def test_registry_from_manifest(tmp_path):
    """load_registry (biasing.py:352-372): one compile per entity file, the
    graph fingerprint attached, duplicate ids and missing files rejected."""
    fst = ab.parse_text_fst(F1_TEXT)
    st = ab.parse_symbol_table("<eps> 0\nalpha 1\nbravo 2\ncharlie 3\n")
    (tmp_path / "e.txt").write_text("alpha bravo\n")
    reg = ab.load_registry(fst, st, [("c1", str(tmp_path / "e.txt"))], ab.BoostCompileConfig())
    assert reg.get("c1").arc_indices.tolist() == [0, 2, 4]
    assert reg.graph_fingerprint == fst.fingerprint()
    with pytest.raises(ab.BiasingCompileError, match="duplicate context id"):
        ab.load_registry(fst, st, [("c1", str(tmp_path / "e.txt"))] * 2, ab.BoostCompileConfig())
    with pytest.raises(ab.BiasingCompileError, match="cannot read entity file"):
        ab.load_registry(fst, st, [("c1", str(tmp_path / "none.txt"))], ab.BoostCompileConfig())


def test_unloadable_scores_are_per_utterance_errors(tmp_path):
    """harness.py:205-219: a score file that fails to load is that
    utterance's error (no decode runs, so no device is needed)."""
    csr = ab.build_csr(ab.parse_text_fst(F1_TEXT))
    st = ab.parse_symbol_table("<eps> 0\nalpha 1\nbravo 2\ncharlie 3\n")
    (tmp_path / "bad.scores").write_text("1 3 0.03\n0 0\n")
    specs = H.read_utterance_specs(f"u1\tch\t{tmp_path}/nope.scores\t-\talpha\n"
                                   f"u2\tch2\t{tmp_path}/bad.scores\n")
    report, jsonl = H.run_decode(csr, st, None, specs, ab.DecoderConfig())
    assert jsonl == []
    assert report.utterances[0]["error"].startswith("FileNotFoundError: [Errno 2]")
    assert report.utterances[1]["error"].startswith("ScoreFormatError:")
    assert report.wer is None and report.rtfx is None and report.biasing == "none"


# ------------------------------------------------------------------ run_decode on the device

def materialise(case, d):
    for fn, text in {**case["entity_files"], **case["score_files"]}.items():
        (d / fn).write_text(text, encoding="utf-8")
    csr = parse_text_fst_csr(case["graph"])  # native ingest (row f2)
    st = ab.parse_symbol_table(case["symtab"])
    registry = None
    if case["biased"]:
        manifest = "".join(f"{fn.rsplit('.', 1)[0]}\t{d / fn}\n" for fn in case["entity_files"])
        registry = ab.load_registry(csr, st, ab.read_context_manifest(manifest), ab.BoostCompileConfig())
    specs = H.read_utterance_specs(case["manifest"].replace("{dir}", str(d)))
    return csr, st, registry, specs


@pytest.mark.gpu
def test_run_decode_matches_reference(golden, tmp_path):
    for case in golden["runs"]:
        d = tmp_path / case["name"]
        d.mkdir()
        csr, st, registry, specs = materialise(case, d)
        report, jsonl = H.run_decode(csr, st, registry, specs, ab.DecoderConfig(**case["cfg"]))
        got = json.loads(report.to_json().replace(str(d), "{dir}"))
        assert set(got["timing"]) == {"load_s", "decode_s", "score_s", "wall_s"}
        del got["timing"]
        got["rtfx"] = got["rtfx"] is not None
        assert got == case["report"], case["name"]
        assert [line.replace(str(d), "{dir}") for line in jsonl] == case["jsonl"], case["name"]
