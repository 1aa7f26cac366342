"""Acoustic cost rows (reference scores.py:19-49): ``costs[t, j]`` is the cost
of emitting input label ``j + 1`` at frame ``t``, added to path costs as-is."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class ScoreFormatError(ValueError):
    """Malformed score matrix."""


@dataclass
class ScoreMatrix:
    costs: np.ndarray
    frame_duration: float = 0.03

    def __post_init__(self) -> None:
        c = np.asarray(self.costs)
        if c.dtype != np.float32:
            c = np.asarray(c, dtype=np.float64)
        if c.ndim != 2:
            raise ScoreFormatError("score matrix must be 2-dimensional")
        if not np.all(np.isfinite(c)):
            raise ScoreFormatError("score matrix contains non-finite costs")
        if self.frame_duration <= 0:
            raise ScoreFormatError("frame_duration must be positive")
        self.costs = c

    @property
    def num_frames(self) -> int:
        return self.costs.shape[0]

    @property
    def num_ilabels(self) -> int:
        return self.costs.shape[1]

    @property
    def audio_seconds(self) -> float:
        return self.num_frames * self.frame_duration

    def row(self, frame: int) -> np.ndarray:
        return self.costs[frame]


def parse_score_matrix(text: str | bytes) -> ScoreMatrix:
    """The reference's score-matrix text format (scores.py:52-80), parsed
    natively: header ``num_frames num_ilabels frame_duration`` then one cost
    row per frame; same checks and ScoreFormatError messages."""
    import ctypes as C

    from . import _lib

    data = text.encode() if isinstance(text, str) else bytes(text)
    lib = _lib.load()
    h = C.c_void_p()
    rc = lib.ab_scores_parse(data, len(data), C.byref(h))
    if rc == _lib.AB_ERR_SCORE_FORMAT:
        raise ScoreFormatError(lib.ab_last_error().decode("utf-8", "replace"))
    if rc == _lib.AB_ERR_INVALID:
        raise ValueError(lib.ab_last_error().decode("utf-8", "replace"))
    _lib.check(rc)
    try:
        T = C.c_int64()
        L = C.c_int64()
        dur = C.c_double()
        _lib.check(lib.ab_scores_info(h, C.byref(T), C.byref(L), C.byref(dur)))
        costs = np.empty((T.value, L.value), dtype=np.float64)
        _lib.check(lib.ab_scores_copy(h, costs.ctypes.data))
    finally:
        lib.ab_scores_destroy(h)
    return ScoreMatrix(costs=costs, frame_duration=dur.value)


def load_score_matrix(path) -> ScoreMatrix:
    """scores.py:91-92: a score-matrix text file."""
    from pathlib import Path

    return parse_score_matrix(Path(path).read_bytes())
