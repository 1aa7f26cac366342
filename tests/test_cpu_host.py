"""CPU tests: the C-ABI library loads and exports every symbol the header
declares; host-side logic (lifecycle checks, contexts, graph types, synthetic
inputs) behaves like the reference.  No compute calls without a GPU."""

import ctypes
import hashlib
import json
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import F1_TEXT, GOLDEN, ROOT

import paper_2306_15685_b200 as ab
from paper_2306_15685_b200 import _lib


def header_symbols():
    text = (ROOT / "include" / "arcboost_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(ab_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 18
    lib = _lib.load()
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_lib.SIGNATURES) == syms


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_header():
    # sizes of the C structs (include/arcboost_b200.h) as seen by ctypes
    assert ctypes.sizeof(_lib.ab_config) == 32
    assert ctypes.sizeof(_lib.ab_capacity) == 32
    assert ctypes.sizeof(_lib.ab_hyp) == 48
    assert ctypes.sizeof(_lib.ab_channel_info) == 96


def test_device_count_call_is_safe_without_gpu():
    n = ctypes.c_int32(-1)
    _lib.load().ab_device_count(ctypes.byref(n))
    assert n.value >= 0


def test_decoder_config_validation():
    with pytest.raises(ValueError):
        ab.DecoderConfig(beam=0)
    with pytest.raises(ValueError):
        ab.DecoderConfig(max_active=0)
    with pytest.raises(ValueError):
        ab.DecoderConfig(partial_every=0)


def test_lifecycle_checks_on_host():
    cfg = ab.DecoderConfig()
    ctx = ab.BiasingContext("c1", np.array([0, 2, 4]), -2.0)
    reg = ab.ContextRegistry({"c1": ctx}, graph_fingerprint="")
    with pytest.raises(ab.UnknownContextError):
        ab.init_channel("c", reg, "missing", cfg)
    with pytest.raises(ab.DecodeError):
        ab.init_channel("c", None, "c1", cfg)
    ch = ab.init_channel("c", reg, None, cfg)
    ab.switch_context(ch, reg, "c1")
    assert ch.context_id == "c1"
    with pytest.raises(ab.UnknownContextError):
        ab.switch_context(ch, reg, "ghost")
    ch.status = ab.ChannelStatus.DECODING
    with pytest.raises(ab.DecodeError, match="mid-utterance"):
        ab.switch_context(ch, reg, None)
    ch.status = ab.ChannelStatus.FINISHED
    ab.switch_context(ch, reg, None)
    assert ch.status is ab.ChannelStatus.IDLE and ch.context_id is None
    # fresh partial needs no device
    h = ab.partial_hypothesis(ab.init_channel("p", None, None, cfg))
    assert h.words == [] and h.cost == 0.0 and h.kind == "partial"
    # finalize of an idle non-fresh channel is rejected before any device call
    ch2 = ab.init_channel("x", None, None, cfg)
    ch2._fresh = False
    csr = ab.build_csr(ab.parse_text_fst(F1_TEXT))
    with pytest.raises(ab.DecodeError):
        ab.finalize(ch2, csr)
    ch3 = ab.init_channel("y", None, None, cfg)
    ch3.status = ab.ChannelStatus.FINISHED
    with pytest.raises(ab.DecodeError, match="cannot advance"):
        ab.advance_frame(ch3, np.zeros(3), csr, None, cfg)


def test_detect_endpoint_thresholds():
    cfg = ab.DecoderConfig(endpoint_silence_frames=20)
    ch = ab.init_channel("c", None, None, cfg)
    ch.trailing_silence = 20
    assert ab.detect_endpoint(ch, cfg)
    ch.trailing_silence = 0
    assert not ab.detect_endpoint(ch, cfg)
    ch.trailing_silence = 1
    assert ab.detect_endpoint(ch, ab.DecoderConfig(endpoint_silence_frames=1))


def test_biasing_context_validation_and_lookup():
    with pytest.raises(ab.BiasingCompileError):
        ab.BiasingContext("x", np.array([3, 1]), -2.0)
    with pytest.raises(ab.BiasingCompileError):
        ab.BiasingContext("x", np.array([-1, 2]), -2.0)
    c = ab.BiasingContext("x", np.array([0, 2, 4]), -2.0)
    assert c.boosted_mask(np.array([0, 1, 2, 3, 4, 5])).tolist() == [1, 0, 1, 0, 1, 0]
    assert ab.effective_weight(c, 2, 0.3) == pytest.approx(-1.7)
    assert ab.effective_weight(c, 1, 0.9) == 0.9
    assert ab.effective_weight(None, 2, 0.3) == 0.3
    d = ab.BiasingContext.from_json_dict(json.loads(c.to_json()))
    assert d.arc_indices.tolist() == [0, 2, 4] and d.discount == -2.0


def test_csr_layout_and_fingerprint_match_reference():
    csr = ab.build_csr(ab.parse_text_fst(F1_TEXT))
    # reference tests/test_fst.py:83-87
    assert csr.row_offsets.tolist() == [0, 2, 4, 4, 5]
    assert csr.weights.tolist() == [0.5, 0.9, 0.3, 0.1, 0.7]
    assert csr.num_emitting_labels == 3
    # the reference's F1 fingerprint (fst.py:194-201 digest over the same text)
    h = hashlib.sha256()
    h.update(b"0 4\n")
    for line in ["1 1 1 0.5", "3 3 3 0.9", "2 2 2 0.3", "0 0 3 0.1", "2 2 2 0.7"]:
        h.update((line + "\n").encode())
    h.update(b"f 2 0.0\nf 3 0.4\n")
    assert csr.fingerprint == h.hexdigest()


def test_benchmark_graph_matches_reference_arrays():
    """synth.benchmark_graph draws the same arrays as the reference's
    build_benchmark_graph (digest recorded by tests/golden/make_golden.py)."""
    from paper_2306_15685_b200 import synth

    want = json.loads((GOLDEN / "graph_digest.json").read_text())
    csr = synth.benchmark_graph(10_000, 4, 2000, seed=421)
    h = hashlib.sha256()
    for a, dt in ((csr.row_offsets, np.int64), (csr.ilabels, np.int64), (csr.olabels, np.int64),
                  (csr.next_states, np.int64), (csr.weights, np.float64)):
        h.update(np.ascontiguousarray(a, dtype=dt).tobytes())
    assert h.hexdigest() == want["g_small"]
    assert csr.num_arcs == want["num_arcs"]
    assert len(csr.finals) == 10_000 and csr.finals[9_999] == 0.0


def test_unigram_context_is_olabel_set():
    from paper_2306_15685_b200 import synth

    csr = synth.benchmark_graph(10_000, 4, 2000, seed=421)
    ctx = synth.unigram_context(csr, 20, 1, num_labels=2000)
    g = json.loads((GOLDEN / "c1_small.json").read_text())
    assert ctx.arc_indices.tolist() == g["ctx_arcs"]
    assert len(ctx.arc_indices) > 0
