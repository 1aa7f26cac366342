"""ctypes binding of the C ABI in include/arcboost_b200.h.

The shared library is built in-tree (``python -c "import __graft_entry__ as g;
g.build()"`` or ``make -C paper_2306_15685_b200``).  There is no fallback: if
the library is missing the import fails loudly.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_NAME = "libarcboost_b200.so"
LIB_PATH = PKG_DIR / LIB_NAME

AB_OK = 0
AB_ERR_INVALID = 1
AB_ERR_CUDA = 2
AB_ERR_DEAD = 3
AB_ERR_STATUS = 4
AB_ERR_CAPACITY = 5
AB_ERR_UNKNOWN_CTX = 6
AB_ERR_WIDTH = 7
AB_ERR_PARSE = 8
AB_ERR_STRUCTURE = 9
AB_ERR_SCORE_FORMAT = 10

AB_IDLE, AB_DECODING, AB_ENDPOINTED, AB_FINISHED = 0, 1, 2, 3
AB_PARTIAL, AB_FINAL = 0, 1
AB_F32, AB_F64 = 0, 1
AB_MODE_ADVANCE, AB_MODE_STREAM = 0, 1
AB_CFG_EXACT = 1
AB_CTX_AUTO, AB_CTX_LIST, AB_CTX_BITSET, AB_CTX_LABELS = 0, 1, 2, 3
AB_MAX_TOKENS, AB_MAX_HASH_SLOTS, AB_MAX_EPSILON_ROUNDS = 131072, 4194304, 2147483647


class ab_config(C.Structure):
    _fields_ = [
        ("beam", C.c_double),
        ("max_active", C.c_int32),
        ("max_epsilon_expansion", C.c_int32),
        ("partial_every", C.c_int32),
        ("endpoint_silence_frames", C.c_int32),
        ("silence_ilabel", C.c_int32),
        ("flags", C.c_int32),
    ]


class ab_capacity(C.Structure):
    _fields_ = [
        ("table_slots", C.c_int64),
        ("frontier_rows", C.c_int64),
        ("arena_records", C.c_int64),
        ("path_words", C.c_int64),
    ]


class ab_channel_info(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("fresh", C.c_int32),
        ("frame_index", C.c_int64),
        ("total_frames", C.c_int64),
        ("utterance_index", C.c_int64),
        ("trailing_silence", C.c_int64),
        ("eps_truncations", C.c_int64),
        ("context", C.c_int32),
        ("num_active", C.c_int32),
        ("store_len", C.c_int64),
        ("error", C.c_int32),
        ("cut_redos", C.c_int32),
        ("tok_expansions", C.c_uint64),
        ("emit_arcs", C.c_uint64),
        ("eps_arcs", C.c_uint64),
    ]


class ab_hyp(C.Structure):
    _fields_ = [
        ("cost", C.c_double),
        ("frame", C.c_int64),
        ("kind", C.c_int32),
        ("fallback", C.c_int32),
        ("hits", C.c_int32),
        ("shared", C.c_int32),
        ("n_words", C.c_int32),
        ("pad_", C.c_int32),
        ("words_off", C.c_int64),
    ]


class ab_decode_args(C.Structure):
    _fields_ = [
        ("n", C.c_int32),
        ("channels", C.c_void_p),
        ("frames", C.c_void_p),
        ("score_offsets", C.c_void_p),
        ("scores", C.c_void_p),
        ("scores_on_device", C.c_int32),
        ("scores_dtype", C.c_int32),
        ("width", C.c_int32),
        ("mode", C.c_int32),
        ("config", ab_config),
        ("stream", C.c_void_p),
    ]


# every symbol the header declares: (name, restype, argtypes)
_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
SIGNATURES = {
    "ab_last_error": (C.c_char_p, []),
    "ab_device_count": (_I32, [C.POINTER(_I32)]),
    "ab_reload_env": (None, []),
    "ab_graph_create": (_I32, [_I32, _I32, _I32, _I64, _P, _P, _P, _P, _P, _I32, _P, _P,
                               C.POINTER(_P)]),
    "ab_graph_destroy": (None, [_P]),
    "ab_graph_query": (_I32, [_P, C.POINTER(_I32), C.POINTER(_I32), C.POINTER(_I64)]),
    "ab_context_register": (_I32, [_P, _P, _I64, C.c_double, _I32, C.POINTER(_I32)]),
    "ab_context_release": (_I32, [_P, _I32]),
    "ab_context_mode": (_I32, [_P, _I32, C.POINTER(_I32)]),
    "ab_context_slack": (_I32, [_P, _I32, C.POINTER(C.c_double), C.POINTER(_I32)]),
    "ab_decoder_create": (_I32, [_P, C.POINTER(ab_capacity), _I32, C.POINTER(_P)]),
    "ab_decoder_destroy": (None, [_P]),
    "ab_decoder_query": (_I32, [_P, C.POINTER(ab_capacity), C.POINTER(_I64)]),
    "ab_channel_init": (_I32, [_P, _I32, _I32]),
    "ab_channel_set_context": (_I32, [_P, _I32, _I32]),
    "ab_channel_get": (_I32, [_P, _I32, C.POINTER(ab_channel_info)]),
    "ab_channel_put": (_I32, [_P, _I32, C.POINTER(ab_channel_info)]),
    "ab_channel_tokens": (_I32, [_P, _I32, _P, _P, _P, _P, _I32, C.POINTER(_I32)]),
    "ab_decode": (_I32, [_P, C.POINTER(ab_decode_args)]),
    "ab_read_results": (_I32, [_P, _P, _P, _P, _I32, _P, _I64, C.POINTER(_I64)]),
    "ab_partial": (_I32, [_P, _I32, C.POINTER(ab_hyp), _P, _I32]),
    "ab_finalize": (_I32, [_P, _I32, C.POINTER(ab_hyp), _P, _I32]),
    "ab_last_kernel_ms": (_I32, [_P, C.POINTER(C.c_float)]),
    "ab_last_launch_count": (_I32, [_P, C.POINTER(_I32)]),
    "ab_channels_init": (_I32, [_P, _I32, _P, _P]),
    "ab_channels_set_context": (_I32, [_P, _I32, _P, _P]),
    "ab_channels_get": (_I32, [_P, _I32, _P, _P]),
    "ab_fst_parse": (_I32, [C.c_char_p, _I64, _I64, C.POINTER(_P)]),
    "ab_fst_load": (_I32, [C.c_char_p, _I64, _I32, C.c_char_p, C.POINTER(_I32), C.POINTER(_P)]),
    "ab_fst_info": (_I32, [_P, C.POINTER(_I32), C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I32),
                           C.c_char_p]),
    "ab_fst_arrays": (_I32, [_P, _P, _P, _P, _P, _P, _P, _P]),
    "ab_fst_destroy": (None, [_P]),
    "ab_graph_create_from_fst": (_I32, [_I32, _P, C.POINTER(_P)]),
    "ab_scores_parse": (_I32, [C.c_char_p, _I64, C.POINTER(_P)]),
    "ab_scores_info": (_I32, [_P, C.POINTER(_I64), C.POINTER(_I64), C.POINTER(C.c_double)]),
    "ab_scores_copy": (_I32, [_P, _P]),
    "ab_scores_destroy": (None, [_P]),
    "ab_compile_context": (_I32, [_I32, _I64, _P, _P, _P, _I32, _P, _P, _I32, _I32, _P, _I64,
                                  C.POINTER(_I64), _P]),
    "ab_align": (_I32, [_P, _I64, _P, _I64, _P, _P, _P, _I64, C.POINTER(_I64)]),
    "ab_edit_distances": (_I32, [_I64, _P, _P, _P, _P, _I32, _P]),
    "ab_scores_generate": (_I32, [_I32, _P, _I32, _I64, C.c_double, C.c_double, C.c_double, _I32, _P, _P]),
}

_lib = None


class AbError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def load() -> C.CDLL:
    """Load the in-tree CUDA library; raises ImportError if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("ARCBOOST_B200_LIB", str(LIB_PATH))
    if not os.path.exists(path):
        raise ImportError(
            f"{LIB_NAME} not found at {path}: build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)"
        )
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != AB_OK:
        msg = load().ab_last_error().decode("utf-8", "replace")
        raise AbError(rc, msg)
