"""Paper Alg. 1: compile word-sequence entities into the arc indices a biasing
context boosts (reference biasing.py:174-285: ``states_that_output_token``,
``dfs_special``, ``find_boost_arcs``, ``compile_context``).

The graph walk runs natively (``ab_compile_context`` in the C ABI, C++ over
the host CSR, one thread per entity batch share); this module keeps the
reference's names, arguments, errors and statistics.  Graphs are accepted as
``CsrFst`` (this package's or the reference's) or adjacency-list ``Fst``.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from .biasing import BiasingCompileError, BiasingContext, ContextStats

EPSILON = 0


@dataclass
class BoostCompileConfig:
    """Compile knobs (reference biasing.py:61-73)."""

    discount: float = -2.0
    lm_order: int = 3  # recorded for provenance; traversal depth is bounded separately
    max_epsilon_depth: int = 10
    skip_oov: bool = True
    allow_positive_discount: bool = False

    def __post_init__(self) -> None:
        if self.discount > 0 and not self.allow_positive_discount:
            raise BiasingCompileError(
                f"discount {self.discount} would penalize, not boost; "
                "set allow_positive_discount to override")
        if self.max_epsilon_depth < 0:
            raise BiasingCompileError("max_epsilon_depth must be >= 0")


def csr_arrays(fst) -> tuple[int, np.ndarray, np.ndarray, np.ndarray]:
    """(num_states, row_offsets i64, olabels i32, next_states i32) of a graph."""
    if hasattr(fst, "row_offsets") and hasattr(fst, "olabels"):
        ro = np.ascontiguousarray(fst.row_offsets, dtype=np.int64)
        return (len(ro) - 1, ro, np.ascontiguousarray(fst.olabels, dtype=np.int32),
                np.ascontiguousarray(fst.next_states, dtype=np.int32))
    counts = np.fromiter((len(out) for out in fst.arcs), dtype=np.int64, count=fst.num_states)
    ro = np.zeros(fst.num_states + 1, dtype=np.int64)
    np.cumsum(counts, out=ro[1:])
    ol = np.fromiter((a.olabel for out in fst.arcs for a in out), dtype=np.int32, count=int(ro[-1]))
    ns = np.fromiter((a.next_state for out in fst.arcs for a in out), dtype=np.int32,
                     count=int(ro[-1]))
    return fst.num_states, ro, ol, ns


def _compile(arrays, entities: Sequence[Sequence[int]], depth: int,
             threads: int = 0) -> tuple[np.ndarray, np.ndarray]:
    S, ro, ol, ns = arrays
    off = np.zeros(len(entities) + 1, dtype=np.int64)
    if entities:
        np.cumsum([len(e) for e in entities], out=off[1:])
    labels = np.ascontiguousarray(np.concatenate([np.asarray(e, dtype=np.int32) for e in entities])
                                  if entities and off[-1] else np.zeros(1, dtype=np.int32))
    status = np.zeros(max(len(entities), 1), dtype=np.int32)
    lib = _lib.load()
    n = C.c_int64()
    cap = 1 << 16
    while True:
        out = np.empty(cap, dtype=np.int64)
        _lib.check(lib.ab_compile_context(
            int(S), int(ro[-1]), ro.ctypes.data, ol.ctypes.data, ns.ctypes.data, len(entities),
            off.ctypes.data, labels.ctypes.data, int(depth), int(threads), out.ctypes.data, cap,
            C.byref(n), status.ctypes.data))
        if n.value <= cap:
            return out[:n.value].copy(), status[:len(entities)]
        cap = n.value


def _check_words(words: Sequence[int]) -> None:
    if not len(words):
        raise BiasingCompileError("empty word sequence")
    if any(int(w) == EPSILON for w in words):
        raise BiasingCompileError("epsilon is not a boostable token")


def find_boost_arcs(fst, words: Sequence[int], cfg: BoostCompileConfig) -> list[int]:
    """Global indices of the arcs to boost for one word sequence
    (biasing.py:203-233); empty if the sequence is unmatchable."""
    _check_words(words)
    arcs, _ = _compile(csr_arrays(fst), [list(words)], cfg.max_epsilon_depth, threads=1)
    return arcs.tolist()


def compile_context(fst, symtab, entities, cfg: BoostCompileConfig, id: str,
                    threads: int = 0) -> BiasingContext:
    """Union of find_boost_arcs over all in-vocabulary entities
    (biasing.py:236-285): duplicate entities are compiled once, entities with
    an out-of-vocabulary word are skipped whole and counted (or raise with
    ``skip_oov=False``)."""
    stats = ContextStats()
    seen: set[tuple[str, ...]] = set()
    todo: list[list[int]] = []
    entries = entities.entries if hasattr(entities, "entries") else entities
    for entry in entries:
        key = tuple(entry)
        if key in seen:
            continue
        seen.add(key)
        labels: list[int] = []
        oov_word = None
        for word in entry:
            label = symtab.get_id(word)
            if label is None or label == EPSILON:
                oov_word = word
                break
            labels.append(int(label))
        if oov_word is not None:
            if not cfg.skip_oov:
                raise BiasingCompileError(
                    f"out-of-vocabulary word {oov_word!r} in entity {' '.join(entry)!r}")
            stats.skipped_oov += 1
            continue
        _check_words(labels)
        todo.append(labels)
    if todo:
        arcs, status = _compile(csr_arrays(fst), todo, cfg.max_epsilon_depth,
                                threads or (os.cpu_count() or 1))
        stats.compiled = int((status == 1).sum())
        stats.unmatched = int((status == 0).sum())
    else:
        arcs = np.zeros(0, dtype=np.int64)
    stats.empty = not len(arcs)
    return BiasingContext(id=id, arc_indices=arcs, discount=cfg.discount, stats=stats)
