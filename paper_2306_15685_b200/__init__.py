"""arcboost-b200: batched, lattice-free token-passing Viterbi over a WFST with
per-channel contextual biasing, on NVIDIA B200 (sm_100a).

Drop-in for the decode path of the reference package ``arcboost``
(arcboost/__init__.py:21-35): the decoder and context names below keep the
reference's signatures and error behaviour; the work runs in the CUDA library
``libarcboost_b200.so`` (C ABI in include/arcboost_b200.h).
"""

from .biasing import (
    BiasingCompileError,
    BiasingContext,
    ContextRegistry,
    UnknownContextError,
    effective_weight,
    sorted_contains,
)
from .decoder import (
    Channel,
    ChannelResult,
    ChannelStatus,
    DecodeError,
    DecoderConfig,
    Hypothesis,
    advance_frame,
    decode_batch,
    detect_endpoint,
    finalize,
    init_channel,
    partial_hypothesis,
    switch_context,
)
from .compiler import (
    BoostCompileConfig,
    EntityList,
    compile_context,
    find_boost_arcs,
    load_registry,
    read_context_manifest,
)
from .device import BatchDecoder, Capacity, DeviceGraph, device_graph
from .fst import (
    EPSILON,
    Arc,
    CsrFst,
    Fst,
    SymbolTable,
    SymbolTableError,
    build_csr,
    csr_from_arrays,
    parse_symbol_table,
    parse_text_fst,
)
from .scores import ScoreMatrix
from . import harness, metrics

__all__ = [
    "EPSILON", "Arc", "BatchDecoder", "BiasingCompileError", "BiasingContext", "BoostCompileConfig",
    "Capacity", "EntityList", "SymbolTable", "SymbolTableError", "compile_context", "find_boost_arcs",
    "harness", "load_registry", "metrics", "parse_symbol_table", "read_context_manifest",
    "Channel", "ChannelResult", "ChannelStatus", "ContextRegistry", "CsrFst", "DecodeError",
    "DecoderConfig", "DeviceGraph", "Fst", "Hypothesis", "ScoreMatrix", "UnknownContextError",
    "advance_frame", "build_csr", "csr_from_arrays", "decode_batch", "detect_endpoint",
    "device_graph", "effective_weight", "finalize", "init_channel", "parse_text_fst",
    "partial_hypothesis", "sorted_contains", "switch_context",
]
