"""ctypes wrapper of the C oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module.  It restates the reference decoder
(/root/reference/pkg/src/arcboost/decoder.py) and is the checker the CUDA path
is compared against; it is never the thing measured as the product.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libarcboost_oracle.so"

IDLE, DECODING, ENDPOINTED, FINISHED = 0, 1, 2, 3
OK, ERR_DEAD, ERR_WIDTH, ERR_STATUS, ERR_CAPACITY, ERR_ALLOC = range(6)


class _Graph(C.Structure):
    _fields_ = [
        ("start", C.c_int32),
        ("num_states", C.c_int32),
        ("num_arcs", C.c_int64),
        ("row_offsets", C.c_void_p),
        ("ilabels", C.c_void_p),
        ("olabels", C.c_void_p),
        ("next_states", C.c_void_p),
        ("weights", C.c_void_p),
        ("is_final", C.c_void_p),
        ("final_costs", C.c_void_p),
        ("num_emitting_labels", C.c_int32),
    ]


class _Config(C.Structure):
    _fields_ = [
        ("beam", C.c_double),
        ("max_active", C.c_int32),
        ("max_eps", C.c_int32),
        ("partial_every", C.c_int32),
        ("endpoint_silence_frames", C.c_int32),
        ("silence_ilabel", C.c_int32),
    ]


class _Context(C.Structure):
    _fields_ = [("arc_indices", C.c_void_p), ("k", C.c_int64), ("discount", C.c_double)]


class _Hyp(C.Structure):
    _fields_ = [
        ("cost", C.c_double),
        ("frame", C.c_int64),
        ("kind", C.c_int32),
        ("fallback", C.c_int32),
        ("hits", C.c_int64),
        ("words_off", C.c_int64),
        ("n_words", C.c_int64),
    ]


class _Info(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("fresh", C.c_int32),
        ("frame_index", C.c_int64),
        ("total_frames", C.c_int64),
        ("utterance_index", C.c_int64),
        ("trailing_silence", C.c_int64),
        ("eps_truncations", C.c_int64),
        ("num_active", C.c_int64),
        ("store_len", C.c_int64),
        ("tok_expansions", C.c_int64),
        ("emit_arcs", C.c_int64),
        ("eps_arcs", C.c_int64),
    ]


_lib = None


def build(force: bool = False) -> Path:
    if force or not LIB_PATH.exists() or (
        LIB_PATH.stat().st_mtime < (HERE / "arcboost_oracle.c").stat().st_mtime
    ):
        subprocess.run(["make", "-C", str(HERE)], check=True, capture_output=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        L.orc_channel_new.restype = C.c_void_p
        L.orc_channel_new.argtypes = [C.POINTER(_Graph)]
        L.orc_channel_free.argtypes = [C.c_void_p]
        L.orc_channel_get_info.argtypes = [C.c_void_p, C.POINTER(_Info)]
        L.orc_channel_set_status.argtypes = [C.c_void_p, C.c_int32]
        L.orc_channel_set_trailing_silence.argtypes = [C.c_void_p, C.c_int64]
        L.orc_advance.argtypes = [C.c_void_p, C.POINTER(_Graph), C.POINTER(_Context),
                                  C.POINTER(_Config), C.c_void_p, C.c_int64]
        L.orc_tokens.restype = C.c_int64
        L.orc_tokens.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]
        L.orc_partial.argtypes = [C.c_void_p, C.POINTER(_Hyp), C.c_void_p, C.c_int64]
        L.orc_finalize.argtypes = [C.c_void_p, C.POINTER(_Graph), C.POINTER(_Hyp), C.c_void_p,
                                   C.c_int64]
        L.orc_decode_stream.argtypes = [
            C.c_void_p, C.POINTER(_Graph), C.POINTER(_Context), C.POINTER(_Config), C.c_void_p,
            C.c_int64, C.c_int64, C.POINTER(_Hyp), C.c_int64, C.POINTER(C.c_int64), C.c_void_p,
            C.c_int64, C.POINTER(C.c_int64)]
        _lib = L
    return _lib


@dataclass
class OHyp:
    words: list
    cost: float
    frame: int
    kind: str
    fallback: bool
    hits: int


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__({ERR_DEAD: "no active tokens", ERR_WIDTH: "emitting-label count",
                          ERR_STATUS: "status", ERR_CAPACITY: "capacity",
                          ERR_ALLOC: "alloc"}.get(code, str(code)))
        self.code = code


class OracleGraph:
    """Arrays of a CsrFst (fst.py:116-162); any object with those attributes works."""

    def __init__(self, start, row_offsets, ilabels, olabels, next_states, weights, finals):
        self.row_offsets = np.ascontiguousarray(row_offsets, dtype=np.int64)
        self.ilabels = np.ascontiguousarray(ilabels, dtype=np.int32)
        self.olabels = np.ascontiguousarray(olabels, dtype=np.int32)
        self.next_states = np.ascontiguousarray(next_states, dtype=np.int32)
        self.weights = np.ascontiguousarray(weights, dtype=np.float64)
        n = len(self.row_offsets) - 1
        self.num_states = n
        self.is_final = np.zeros(max(n, 1), dtype=np.uint8)
        self.final_costs = np.zeros(max(n, 1), dtype=np.float64)
        if hasattr(finals, "as_arrays"):
            fs, fc = finals.as_arrays()
            self.is_final[np.asarray(fs)] = 1
            self.final_costs[np.asarray(fs)] = np.asarray(fc, dtype=np.float64)
        elif isinstance(finals, dict):
            for s, w in finals.items():
                self.is_final[int(s)] = 1
                self.final_costs[int(s)] = float(w)
        else:
            mask, costs = finals
            self.is_final[:n] = np.asarray(mask, dtype=np.uint8)
            self.final_costs[:n] = np.asarray(costs, dtype=np.float64)
        self.num_emitting_labels = int(self.ilabels.max()) if len(self.ilabels) else 0
        self.c = _Graph(int(start), n, int(self.row_offsets[-1]) if n >= 0 else 0,
                        self.row_offsets.ctypes.data, self.ilabels.ctypes.data,
                        self.olabels.ctypes.data, self.next_states.ctypes.data,
                        self.weights.ctypes.data, self.is_final.ctypes.data,
                        self.final_costs.ctypes.data, self.num_emitting_labels)

    @classmethod
    def from_csr(cls, csr) -> "OracleGraph":
        return cls(csr.start, csr.row_offsets, csr.ilabels, csr.olabels, csr.next_states,
                   csr.weights, csr.finals)


def make_config(cfg) -> _Config:
    return _Config(float(cfg.beam), int(cfg.max_active), int(cfg.max_epsilon_expansion),
                   int(cfg.partial_every), int(cfg.endpoint_silence_frames),
                   int(cfg.silence_ilabel))


class _Ctx:
    def __init__(self, ctx):
        if ctx is None:
            self.ptr = None
            return
        self.idx = np.ascontiguousarray(ctx.arc_indices, dtype=np.int64)
        self.c = _Context(self.idx.ctypes.data, len(self.idx), float(ctx.discount))
        self.ptr = C.byref(self.c)


class OracleChannel:
    def __init__(self, graph: OracleGraph):
        self.graph = graph
        self.h = lib().orc_channel_new(C.byref(graph.c))
        if not self.h:
            raise MemoryError("oracle channel allocation failed")

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib is not None:
            _lib.orc_channel_free(h)
            self.h = None

    def info(self) -> dict:
        i = _Info()
        lib().orc_channel_get_info(self.h, C.byref(i))
        return {f: getattr(i, f) for f, _ in _Info._fields_}

    def set_status(self, s: int) -> None:
        lib().orc_channel_set_status(self.h, s)

    def advance(self, row, ctx, cfg) -> None:
        row = np.ascontiguousarray(row, dtype=np.float64)
        c = _Ctx(ctx)
        rc = lib().orc_advance(self.h, C.byref(self.graph.c), c.ptr, C.byref(make_config(cfg)),
                               row.ctypes.data, len(row))
        if rc:
            raise OracleError(rc)

    def tokens(self):
        n = lib().orc_tokens(self.h, None, None, None, 0)
        st = np.zeros(n, dtype=np.int32)
        co = np.zeros(n, dtype=np.float64)
        hi = np.zeros(n, dtype=np.int64)
        lib().orc_tokens(self.h, st.ctypes.data, co.ctypes.data, hi.ctypes.data, n)
        return st, co, hi

    def _hyp(self, fn, *args) -> OHyp:
        cap = 1 << 20
        words = np.zeros(cap, dtype=np.int32)
        h = _Hyp()
        rc = fn(self.h, *args, C.byref(h), words.ctypes.data, cap)
        if rc:
            raise OracleError(rc)
        return OHyp(words[: h.n_words].tolist(), h.cost, h.frame,
                    "final" if h.kind == 1 else "partial", bool(h.fallback), h.hits)

    def partial(self) -> OHyp:
        return self._hyp(lib().orc_partial)

    def finalize(self) -> OHyp:
        return self._hyp(lib().orc_finalize, C.byref(self.graph.c))


def decode_stream(graph: OracleGraph, scores, ctx, cfg, channel: OracleChannel | None = None,
                  words_cap: int | None = None):
    """_decode_one over one [T, L] matrix. Returns (list[OHyp], error_code)."""
    scores = np.ascontiguousarray(scores, dtype=np.float64)
    T = scores.shape[0]
    width = scores.shape[1] if scores.ndim == 2 else 0
    ch = channel or OracleChannel(graph)
    c = _Ctx(ctx)
    hyp_cap = 2 * T + 2
    if words_cap is None:
        words_cap = max(1 << 16, (T + 2) * (T + 2) * 4)
    hyps = (_Hyp * hyp_cap)()
    words = np.zeros(words_cap, dtype=np.int32)
    nh = C.c_int64(0)
    nw = C.c_int64(0)
    rc = lib().orc_decode_stream(ch.h, C.byref(graph.c), c.ptr, C.byref(make_config(cfg)),
                                 scores.ctypes.data, T, width, hyps, hyp_cap, C.byref(nh),
                                 words.ctypes.data, words_cap, C.byref(nw))
    out = []
    for i in range(nh.value):
        h = hyps[i]
        out.append(OHyp(words[h.words_off:h.words_off + h.n_words].tolist(), h.cost, h.frame,
                        "final" if h.kind == 1 else "partial", bool(h.fallback), h.hits))
    return out, rc
