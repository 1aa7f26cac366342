"""Graph ingest: the native text parser (ab_fst_parse /
ab_fst_load) against the reference's parse_text_fst + build_csr +
fingerprint (tests/golden/fst_cases.json, from tests/golden/make_fst_golden.py):
identical CSR arrays, finals, fingerprints, error types and messages; the
binary cache round-trips.  CPU only."""

import numpy as np
import pytest

from conftest import F1_TEXT, fx, load_json

import paper_2306_15685_b200 as ab
from paper_2306_15685_b200 import fst as M


@pytest.fixture(scope="module")
def cases():
    return load_json("fst_cases.json")


def _check(csr, e):
    assert csr.start == e["start"]
    assert csr.row_offsets.tolist() == e["row_offsets"]
    assert csr.ilabels.tolist() == e["ilabels"]
    assert csr.olabels.tolist() == e["olabels"]
    assert csr.next_states.tolist() == e["next_states"]
    assert [float(w).hex() for w in csr.weights] == e["weights"]
    assert sorted(csr.finals.items()) == [(s, fx(c)) for s, c in e["finals"]]
    assert csr.fingerprint == e["fingerprint"]


def test_texts_match_reference(cases):
    for i, c in enumerate(cases["ok"]):
        _check(M.parse_text_fst_csr(c["text"], c["hint"]), c["expect"])


def test_errors_match_reference(cases):
    for c in cases["errors"]:
        exc = M.FstParseError if c["type"] == "FstParseError" else M.FstStructureError
        with pytest.raises(exc) as ei:
            M.parse_text_fst_csr(c["text"], c["hint"])
        assert str(ei.value) == c["message"]


def test_fingerprint_matches_python_digest():
    csr = M.parse_text_fst_csr(F1_TEXT)
    assert csr.fingerprint == ab.build_csr(ab.parse_text_fst(F1_TEXT)).fingerprint
    assert csr.row_offsets.tolist() == [0, 2, 4, 4, 5]  # tests/test_fst.py:83-87
    assert csr.weights.tolist() == [0.5, 0.9, 0.3, 0.1, 0.7]


def test_file_load_and_binary_cache(tmp_path, cases):
    c = cases["ok"][7]
    p = tmp_path / "g.fst.txt"
    p.write_text(c["text"])
    a = M.load_fst(p, cache=True)
    assert not a.cache_hit and (tmp_path / "g.fst.txt.abcsr").exists()
    b = M.load_fst(p, cache=True)
    assert b.cache_hit
    for csr in (a, b):
        if c["hint"] is None:
            _check(csr, c["expect"])
    # a changed source invalidates the cache
    p.write_text(c["text"] + "# edited\n")
    assert not M.load_fst(p, cache=True).cache_hit


def test_ingested_graph_feeds_the_compiler():
    csr = M.parse_text_fst_csr(F1_TEXT)
    assert ab.find_boost_arcs(csr, [1, 2], ab.BoostCompileConfig()) == [0, 2, 4]


def _bench_text(states):
    from paper_2306_15685_b200 import synth

    csr = synth.benchmark_graph(states, 4, 2000, seed=421, f32_weights=True)
    src = np.repeat(np.arange(csr.num_states), np.diff(csr.row_offsets))
    lines = [f"{a} {b} {c} {d} {w!r}" for a, b, c, d, w in
             zip(src.tolist(), csr.next_states.tolist(), csr.ilabels.tolist(), csr.olabels.tolist(),
                 csr.weights.tolist())]
    lines += [f"{s} {c!r}" for s, c in sorted(csr.finals.items())]
    return csr, "\n".join(lines) + "\n"


def test_large_text_chunked_parse_matches_python():
    """Texts over 4 MB are parsed in parallel chunks: same arrays, same
    fingerprint as the Python path; an error in a late chunk reports the
    same line as a sequential parse."""
    csr, text = _bench_text(60_000)
    assert len(text) > (1 << 22)
    got = M.parse_text_fst_csr(text)
    for k in ("row_offsets", "ilabels", "olabels", "next_states", "weights"):
        assert np.array_equal(getattr(got, k), getattr(csr, k)), k
    finals = dict(csr.finals.items())
    assert got.finals == finals
    assert got.fingerprint == ab.fst.graph_fingerprint(
        csr.start, csr.num_states,
        zip(csr.ilabels.tolist(), csr.olabels.tolist(), csr.next_states.tolist(), csr.weights.tolist()),
        finals)
    lines = text.splitlines()
    bad = len(lines) - 1000
    lines[bad] = "7 8 x 9"
    with pytest.raises(M.FstParseError, match=f"^line {bad + 1}: invalid literal"):
        M.parse_text_fst_csr("\n".join(lines) + "\n")
