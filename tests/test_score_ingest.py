"""Score ingest: the native score-matrix parser against
the reference's parse_score_matrix (tests/golden/score_cases.json, from
tests/golden/make_score_golden.py): identical matrices, frame durations,
error types and messages.  CPU only."""

import pytest

from conftest import load_json

from paper_2306_15685_b200 import scores as SC


@pytest.fixture(scope="module")
def cases():
    return load_json("score_cases.json")


def test_matrices_match_reference(cases):
    for i, c in enumerate(cases["ok"]):
        m = SC.parse_score_matrix(c["text"])
        e = c["expect"]
        assert m.costs.shape == (e["frames"], e["labels"]), i
        assert float(m.frame_duration).hex() == e["dur"], i
        assert [[float(x).hex() for x in row] for row in m.costs] == e["costs"], i


def test_errors_match_reference(cases):
    for c in cases["errors"]:
        exc = SC.ScoreFormatError if c["type"] == "ScoreFormatError" else ValueError
        with pytest.raises(exc) as ei:
            SC.parse_score_matrix(c["text"])
        assert str(ei.value) == c["message"], c["text"]


def test_load_from_file_feeds_the_decoder_api(tmp_path, cases):
    p = tmp_path / "u1.scores"
    p.write_text(cases["ok"][10]["text"])
    m = SC.load_score_matrix(p)
    assert m.num_frames == cases["ok"][10]["expect"]["frames"]
    assert m.audio_seconds == pytest.approx(m.num_frames * m.frame_duration)
