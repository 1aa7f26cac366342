"""Biasing contexts: a strictly increasing list of global arc indices plus one
discount (reference biasing.py:86-137) and the registry that maps context ids
to them (biasing.py:320-349).

On the device every registered context becomes an entry of the context store
(shared-memory sorted list for sparse contexts, HBM bitset for dense ones), so
a per-channel context switch is a handle swap.  Compiling entity lists into
arc indices (paper Alg. 1, biasing.py:174-285) is ``compiler.py`` (native);
contexts compiled by the reference (or by any tool) are accepted as-is,
including via ``BiasingContext.from_json_dict``.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np


class BiasingCompileError(ValueError):
    """Invalid context contents (reference biasing.py:23)."""


class UnknownContextError(KeyError):
    """Lookup of a context id that is not in the registry (biasing.py:27)."""


@dataclass
class ContextStats:
    compiled: int = 0
    skipped_oov: int = 0
    unmatched: int = 0
    empty: bool = False


@dataclass
class BiasingContext:
    id: str
    arc_indices: np.ndarray
    discount: float
    stats: ContextStats = field(default_factory=ContextStats)

    def __post_init__(self) -> None:
        idx = np.asarray(self.arc_indices, dtype=np.int64)
        if idx.ndim != 1:
            raise BiasingCompileError("arc_indices must be one-dimensional")
        if len(idx) and not np.all(idx[1:] > idx[:-1]):
            raise BiasingCompileError("arc_indices must be strictly increasing")
        if len(idx) and idx[0] < 0:
            raise BiasingCompileError("negative arc index")
        self.arc_indices = idx

    def is_boosted(self, g: int) -> bool:
        return sorted_contains(self.arc_indices, g)

    def boosted_mask(self, arc_ids: np.ndarray) -> np.ndarray:
        idx = self.arc_indices
        arc_ids = np.asarray(arc_ids, dtype=np.int64)
        if not len(idx):
            return np.zeros(len(arc_ids), dtype=bool)
        pos = np.minimum(np.searchsorted(idx, arc_ids), len(idx) - 1)
        return idx[pos] == arc_ids

    def to_json_dict(self) -> dict:
        return {"id": self.id, "discount": self.discount,
                "arc_indices": [int(g) for g in self.arc_indices],
                "stats": self.stats.__dict__.copy()}

    def to_json(self) -> str:
        return json.dumps(self.to_json_dict(), indent=2)

    @classmethod
    def from_json_dict(cls, d: dict) -> "BiasingContext":
        return cls(id=d["id"], arc_indices=np.asarray(d["arc_indices"], dtype=np.int64),
                   discount=float(d["discount"]), stats=ContextStats(**d.get("stats", {})))


def sorted_contains(indices: Sequence[int] | np.ndarray, g: int) -> bool:
    """Membership by binary search in a sorted unique sequence (biasing.py:140-163)."""
    lo, hi = 0, len(indices)
    while lo < hi:
        mid = (lo + hi) // 2
        v = indices[mid]
        if v == g:
            return True
        if v < g:
            lo = mid + 1
        else:
            hi = mid
    return False


def effective_weight(ctx: BiasingContext | None, g: int, w: float) -> float:
    """Arc weight seen by the decoder (biasing.py:166-171)."""
    if ctx is not None and ctx.is_boosted(g):
        return w + ctx.discount
    return w


@dataclass
class ContextRegistry:
    contexts: dict
    graph_fingerprint: str

    def get(self, context_id: str) -> BiasingContext:
        try:
            return self.contexts[context_id]
        except KeyError:
            raise UnknownContextError(
                f"unknown biasing context {context_id!r}; known: {sorted(self.contexts)}"
            ) from None

    def resolve(self, context_id: str | None) -> BiasingContext | None:
        return None if context_id is None else self.get(context_id)

    def __contains__(self, context_id: str) -> bool:
        return context_id in self.contexts

    def __len__(self) -> int:
        return len(self.contexts)

    def ids(self) -> list[str]:
        return sorted(self.contexts)

    @classmethod
    def empty(cls, fingerprint: str = "") -> "ContextRegistry":
        return cls(contexts={}, graph_fingerprint=fingerprint)
