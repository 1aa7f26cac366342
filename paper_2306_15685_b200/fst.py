"""Graph types consumed by the decode path.

Only what the hot path needs is provided: the CSR layout whose global arc
index space contexts refer to (``CsrFst``, reference fst.py:116-162), its
builder from an adjacency list (``build_csr``, fst.py:165-191), the graph
fingerprint (fst.py:194-201) and a minimal text reader so tests and tools can
state small graphs the way the reference's tests do (fst.py:204-275).  Any
object exposing the ``CsrFst`` attributes (including the reference's own
``arcboost.fst.CsrFst``) is accepted by the decoder.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field
from typing import Iterable

import numpy as np

EPSILON = 0


class FstError(ValueError):
    """Malformed graph input."""


class FstParseError(FstError):
    """Malformed graph or symbol-table text (reference fst.py:24)."""


class FstStructureError(FstError):
    """Structurally invalid graph (reference fst.py:28)."""


@dataclass(frozen=True)
class Arc:
    ilabel: int
    olabel: int
    next_state: int
    weight: float


@dataclass
class Fst:
    """Adjacency list; arc order inside a state fixes the global arc index."""

    start: int
    num_states: int
    arcs: list
    finals: dict

    def __post_init__(self) -> None:
        if len(self.arcs) != self.num_states:
            raise FstError("arc table length != num_states")
        if self.num_states and not 0 <= self.start < self.num_states:
            raise FstError(f"start state {self.start} out of range for {self.num_states} states")
        for s, out in enumerate(self.arcs):
            for a in out:
                if not 0 <= a.next_state < self.num_states:
                    raise FstError(f"arc from state {s} to nonexistent state {a.next_state}")
                if a.ilabel < 0 or a.olabel < 0:
                    raise FstError(f"negative label on arc from state {s}")
                if not math.isfinite(a.weight):
                    raise FstError(f"non-finite weight on arc from state {s}")

    @property
    def num_arcs(self) -> int:
        return sum(len(out) for out in self.arcs)

    def fingerprint(self) -> str:
        return graph_fingerprint(
            self.start, self.num_states,
            ((a.ilabel, a.olabel, a.next_state, a.weight) for out in self.arcs for a in out),
            self.finals)


def graph_fingerprint(start, num_states, arc_tuples, finals) -> str:
    """Same digest as the reference (fst.py:194-201), so a registry compiled
    against a graph by the reference validates against this package's CSR."""
    h = hashlib.sha256()
    h.update(f"{start} {num_states}\n".encode())
    for il, ol, dst, w in arc_tuples:
        h.update(f"{il} {ol} {dst} {w!r}\n".encode())
    for s in sorted(finals):
        h.update(f"f {s} {finals[s]!r}\n".encode())
    return h.hexdigest()


@dataclass
class CsrFst:
    """State-major CSR; the arc at global index g belongs to state s iff
    row_offsets[s] <= g < row_offsets[s + 1] (reference fst.py:116-162)."""

    start: int
    row_offsets: np.ndarray
    ilabels: np.ndarray
    olabels: np.ndarray
    next_states: np.ndarray
    weights: np.ndarray
    finals: dict
    _fingerprint: str | None = field(default=None, repr=False)

    @property
    def num_states(self) -> int:
        return len(self.row_offsets) - 1

    @property
    def num_arcs(self) -> int:
        return int(self.row_offsets[-1])

    @property
    def num_emitting_labels(self) -> int:
        return int(self.ilabels.max()) if len(self.ilabels) else 0

    @property
    def fingerprint(self) -> str:
        # computed lazily: hashing 2e7 arcs in Python takes tens of seconds
        if self._fingerprint is None:
            self._fingerprint = graph_fingerprint(
                self.start, self.num_states,
                zip(self.ilabels.tolist(), self.olabels.tolist(), self.next_states.tolist(),
                    self.weights.tolist()),
                self.finals)
        return self._fingerprint

    @fingerprint.setter
    def fingerprint(self, v: str) -> None:
        self._fingerprint = v

    def arc_range(self, state: int) -> tuple[int, int]:
        return int(self.row_offsets[state]), int(self.row_offsets[state + 1])


def csr_from_arrays(start, row_offsets, ilabels, olabels, next_states, weights, finals,
                    fingerprint: str | None = None) -> CsrFst:
    return CsrFst(
        start=int(start),
        row_offsets=np.ascontiguousarray(row_offsets, dtype=np.int64),
        ilabels=np.ascontiguousarray(ilabels, dtype=np.int64),
        olabels=np.ascontiguousarray(olabels, dtype=np.int64),
        next_states=np.ascontiguousarray(next_states, dtype=np.int64),
        weights=np.ascontiguousarray(weights, dtype=np.float64),
        finals=dict(finals),
        _fingerprint=fingerprint,
    )


def build_csr(fst: Fst) -> CsrFst:
    """Lay the adjacency list out state-major, arc order preserved (fst.py:165-191)."""
    counts = np.array([len(out) for out in fst.arcs], dtype=np.int64)
    offs = np.zeros(fst.num_states + 1, dtype=np.int64)
    np.cumsum(counts, out=offs[1:])
    flat = [a for out in fst.arcs for a in out]
    return CsrFst(
        start=fst.start,
        row_offsets=offs,
        ilabels=np.array([a.ilabel for a in flat], dtype=np.int64),
        olabels=np.array([a.olabel for a in flat], dtype=np.int64),
        next_states=np.array([a.next_state for a in flat], dtype=np.int64),
        weights=np.array([a.weight for a in flat], dtype=np.float64),
        finals=dict(fst.finals),
        _fingerprint=fst.fingerprint(),
    )


def parse_text_fst(text: str | Iterable[str]) -> Fst:
    """OpenFst-style text: ``src dst ilabel olabel [weight]`` arc lines and
    ``state [weight]`` final lines; the first line names the start state."""
    lines = text.splitlines() if isinstance(text, str) else list(text)
    start = None
    arcs_in: list[tuple[int, Arc]] = []
    finals: dict[int, float] = {}
    top = -1
    for n, raw in enumerate(lines, 1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        f = line.split()
        try:
            if len(f) in (4, 5):
                s, d, il, ol = (int(x) for x in f[:4])
                w = float(f[4]) if len(f) == 5 else 0.0
                arcs_in.append((s, Arc(il, ol, d, w)))
                top = max(top, s, d)
            elif len(f) in (1, 2):
                s = int(f[0])
                if s in finals:
                    raise ValueError(f"duplicate final line for state {s}")
                finals[s] = float(f[1]) if len(f) == 2 else 0.0
                top = max(top, s)
            else:
                raise ValueError(f"expected 1, 2, 4 or 5 fields, got {len(f)}")
        except ValueError as exc:
            raise FstError(f"line {n}: {exc}: {raw!r}") from None
        if start is None:
            start = int(f[0])
    if start is None:
        raise FstError("no start state: input contains no arc or final lines")
    adj: list[list[Arc]] = [[] for _ in range(top + 1)]
    for s, a in arcs_in:
        adj[s].append(a)
    return Fst(start=start, num_states=top + 1, arcs=adj, finals=finals)


# --------------------------------------------------------------- native ingest
def _native_fst(handle) -> CsrFst:
    """CsrFst from a native ab_fst handle (the handle is destroyed)."""
    import ctypes as C

    from . import _lib

    lib = _lib.load()
    try:
        start = C.c_int32()
        S = C.c_int64()
        A = C.c_int64()
        nf = C.c_int32()
        fp = C.create_string_buffer(65)
        _lib.check(lib.ab_fst_info(handle, C.byref(start), C.byref(S), C.byref(A), C.byref(nf), fp))
        ro = np.empty(S.value + 1, dtype=np.int64)
        il = np.empty(A.value, dtype=np.int32)
        ol = np.empty(A.value, dtype=np.int32)
        ns = np.empty(A.value, dtype=np.int32)
        w = np.empty(A.value, dtype=np.float64)
        fs = np.empty(nf.value, dtype=np.int32)
        fc = np.empty(nf.value, dtype=np.float64)
        _lib.check(lib.ab_fst_arrays(handle, ro.ctypes.data, il.ctypes.data, ol.ctypes.data,
                                     ns.ctypes.data, w.ctypes.data, fs.ctypes.data, fc.ctypes.data))
    finally:
        lib.ab_fst_destroy(handle)
    return CsrFst(start=start.value, row_offsets=ro, ilabels=il.astype(np.int64),
                  olabels=ol.astype(np.int64), next_states=ns.astype(np.int64), weights=w,
                  finals={int(s): float(c) for s, c in zip(fs, fc)},
                  _fingerprint=fp.value.decode())


def _ingest_call(fn, *args):
    import ctypes as C

    from . import _lib

    h = C.c_void_p()
    rc = fn(*args, C.byref(h))
    if rc == _lib.AB_ERR_PARSE:
        raise FstParseError(_lib.load().ab_last_error().decode("utf-8", "replace"))
    if rc == _lib.AB_ERR_STRUCTURE:
        raise FstStructureError(_lib.load().ab_last_error().decode("utf-8", "replace"))
    _lib.check(rc)
    return h.value


def parse_text_fst_csr(text: str | bytes, num_states_hint: int | None = None) -> CsrFst:
    """parse_text_fst + build_csr (reference fst.py:165-275) natively: the
    state-major CSR and the reference fingerprint straight from the text."""
    from . import _lib

    data = text.encode() if isinstance(text, str) else bytes(text)
    h = _ingest_call(_lib.load().ab_fst_parse, data, len(data),
                     -1 if num_states_hint is None else int(num_states_hint))
    return _native_fst(h)


def load_fst(path, num_states_hint: int | None = None, cache: bool = True,
             cache_path=None) -> CsrFst:
    """Graph file -> CsrFst.  With ``cache`` a binary copy of the CSR is kept
    next to the file (``<path>.abcsr``) and reused while the file's size and
    modification time are unchanged."""
    import ctypes as C
    import os

    from . import _lib

    path = os.fspath(path)
    cp = os.fspath(cache_path) if cache_path is not None else path + ".abcsr"
    hit = C.c_int32()
    h = _ingest_call(_lib.load().ab_fst_load, path.encode(),
                     -1 if num_states_hint is None else int(num_states_hint), 1 if cache else 0,
                     cp.encode(), C.byref(hit))
    csr = _native_fst(h)
    csr.cache_hit = bool(hit.value)
    return csr


class SymbolTableError(ValueError):
    """Invalid symbol table (reference fst.py:32)."""


class SymbolTable:
    """Bijective word <-> label-id map, id 0 is epsilon (reference
    fst.py:334-373); the harness maps hypothesis labels back to words."""

    def __init__(self, word_to_id: dict[str, int]):
        if 0 not in word_to_id.values():
            raise SymbolTableError("missing epsilon entry at id 0")
        self._word_to_id = dict(word_to_id)
        self._id_to_word: dict[int, str] = {}
        for word, label in self._word_to_id.items():
            if label in self._id_to_word:
                raise SymbolTableError(f"duplicate id {label} ({self._id_to_word[label]!r} vs {word!r})")
            self._id_to_word[label] = word

    def __len__(self) -> int:
        return len(self._word_to_id)

    def __contains__(self, word: str) -> bool:
        return word in self._word_to_id

    def id_of(self, word: str) -> int:
        try:
            return self._word_to_id[word]
        except KeyError:
            raise SymbolTableError(f"unknown word {word!r}") from None

    def get_id(self, word: str) -> int | None:
        return self._word_to_id.get(word)

    def word_of(self, label: int) -> str:
        try:
            return self._id_to_word[label]
        except KeyError:
            raise SymbolTableError(f"unknown label id {label}") from None

    def words(self):
        return iter(self._word_to_id)

    @property
    def epsilon_word(self) -> str:
        return self._id_to_word[EPSILON]


def parse_symbol_table(text) -> SymbolTable:
    """``word id`` lines (reference fst.py:376-400): blank and ``#`` lines
    skipped, duplicate words or ids rejected, the reference's messages."""
    if hasattr(text, "read"):
        text = text.read()
    lines = text.splitlines() if isinstance(text, str) else list(text)
    word_to_id: dict[str, int] = {}
    seen_ids: dict[int, str] = {}
    for lineno, raw in enumerate(lines, start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        fields = line.split()
        if len(fields) != 2:
            raise FstParseError(f"line {lineno}: expected 'word id', got {raw!r}")
        word = fields[0]
        try:
            label = int(fields[1])
        except ValueError:
            raise FstParseError(f"line {lineno}: bad id {fields[1]!r}") from None
        if label < 0:
            raise FstParseError(f"line {lineno}: negative id {label}")
        if word in word_to_id:
            raise SymbolTableError(f"duplicate word {word!r}")
        if label in seen_ids:
            raise SymbolTableError(f"duplicate id {label} ({seen_ids[label]!r} vs {word!r})")
        word_to_id[word] = label
        seen_ids[label] = word
    return SymbolTable(word_to_id)
