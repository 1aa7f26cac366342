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
