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
from pathlib import Path
from typing import Iterable, Sequence

import numpy as np

from . import _lib
from .biasing import BiasingCompileError, BiasingContext, ContextRegistry, ContextStats

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
    return _compile_context_arrays(csr_arrays(fst), symtab, entities, cfg, id, threads)


def _compile_context_arrays(arrays, symtab, entities, cfg: BoostCompileConfig, id: str,
                            threads: int = 0) -> BiasingContext:
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
        arcs, status = _compile(arrays, todo, cfg.max_epsilon_depth,
                                threads or (os.cpu_count() or 1))
        stats.compiled = int((status == 1).sum())
        stats.unmatched = int((status == 0).sum())
    else:
        arcs = np.zeros(0, dtype=np.int64)
    stats.empty = not len(arcs)
    return BiasingContext(id=id, arc_indices=arcs, discount=cfg.discount, stats=stats)


@dataclass
class EntityList:
    """Ordered word sequences to boost (reference biasing.py:31-57)."""

    entries: list[list[str]]
    source: str = ""

    def __post_init__(self) -> None:
        for entry in self.entries:
            if not entry:
                raise BiasingCompileError(f"empty entity in {self.source or 'entity list'}")

    @classmethod
    def parse_text(cls, text: str, source: str = "") -> "EntityList":
        """One entity per line, words space-separated; '#' lines are comments."""
        entries = []
        for raw in text.splitlines():
            line = raw.strip()
            if not line or line.startswith("#"):
                continue
            entries.append(line.split())
        return cls(entries=entries, source=source)

    @classmethod
    def from_file(cls, path) -> "EntityList":
        path = Path(path)
        return cls.parse_text(path.read_text(encoding="utf-8"), source=str(path))


def _graph_fingerprint(fst) -> str:
    fp = getattr(fst, "fingerprint", "")
    return fp() if callable(fp) else fp


def load_registry(fst, symtab, manifest: Iterable[tuple[str, str]], cfg: BoostCompileConfig,
                  threads: int = 0) -> ContextRegistry:
    """Compile every manifest entry before decoding (reference
    biasing.py:352-372): duplicate ids and unreadable entity files raise
    BiasingCompileError; the registry carries the graph fingerprint."""
    contexts: dict[str, BiasingContext] = {}
    arrays = None
    for context_id, path in manifest:
        if context_id in contexts:
            raise BiasingCompileError(f"duplicate context id {context_id!r} in manifest")
        try:
            entities = EntityList.from_file(path)
        except OSError as exc:
            raise BiasingCompileError(f"cannot read entity file {path}: {exc}") from None
        if arrays is None:
            arrays = csr_arrays(fst)
        contexts[context_id] = _compile_context_arrays(arrays, symtab, entities, cfg, context_id, threads)
    return ContextRegistry(contexts=contexts, graph_fingerprint=_graph_fingerprint(fst))


def read_context_manifest(text: str) -> list[tuple[str, str]]:
    """TSV lines ``id<TAB>entity-file-path`` (reference biasing.py:375-389)."""
    rows: list[tuple[str, str]] = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        parts = line.split("\t")
        if len(parts) != 2:
            raise BiasingCompileError(f"manifest line {lineno}: expected 'id<TAB>path', got {raw!r}")
        rows.append((parts[0], parts[1]))
    return rows
