"""Synthetic inputs for the BASELINE configs.

``benchmark_graph`` reproduces the reference's ``build_benchmark_graph``
(arcboost/synth.py:294-322) draw for draw, but returns the CSR arrays directly
(vectorised; the reference builds Python Arc objects, which does not scale to
2e7 arcs).  tests/test_cpu_host.py (test_benchmark_graph_matches_reference)
pins the arrays against the reference's digest.
With ``f32_weights`` the weights are rounded once to float32 so the device can
store 4-byte weights while accumulating bit-exactly in f64; the same rounded
arrays are what the CPU oracle sees.
"""

from __future__ import annotations

import random

import numpy as np

from .biasing import BiasingContext
from .fst import CsrFst, csr_from_arrays


def benchmark_graph(num_states: int, arcs_per_state: int, num_labels: int, *,
                    eps_input_frac: float = 0.1, seed: int = 421,
                    f32_weights: bool = False) -> CsrFst:
    rng = np.random.default_rng(seed)
    n = num_states * arcs_per_state
    dsts = rng.integers(0, num_states, size=n)
    ilabels = rng.integers(1, num_labels + 1, size=n)
    eps_in = rng.random(n) < eps_input_frac
    ilabels[eps_in] = 0
    olabels = rng.integers(0, num_labels + 1, size=n)
    weights = rng.uniform(0.0, 3.0, size=n)
    ilabels[:num_labels] = np.arange(1, num_labels + 1)
    if f32_weights:
        weights = weights.astype(np.float32).astype(np.float64)
    row_offsets = np.arange(0, n + 1, arcs_per_state, dtype=np.int64)
    finals = (np.arange(num_states, dtype=np.int64), np.zeros(num_states))
    csr = csr_from_arrays(0, row_offsets, ilabels, olabels, dsts, weights, {})
    csr.finals = _AllFinal(num_states)
    return csr


class _AllFinal(dict):
    """finals = {s: 0.0 for every state} without materialising 5e6 dict entries
    until someone iterates it (the device upload uses the array form)."""

    def __init__(self, n: int):
        super().__init__()
        self._n = n
        self._filled = False

    def _fill(self):
        if not self._filled:
            super().update({s: 0.0 for s in range(self._n)})
            self._filled = True

    def as_arrays(self):
        return np.arange(self._n, dtype=np.int32), np.zeros(self._n, dtype=np.float64)

    def __len__(self):
        return self._n

    def __contains__(self, s):
        return 0 <= int(s) < self._n

    def __getitem__(self, s):
        if s in self:
            return 0.0
        raise KeyError(s)

    def get(self, s, default=None):
        return 0.0 if s in self else default

    def __iter__(self):
        return iter(range(self._n))

    def keys(self):
        return range(self._n)

    def values(self):
        return (0.0 for _ in range(self._n))

    def items(self):
        return ((s, 0.0) for s in range(self._n))

    def copy(self):
        self._fill()
        return dict(self)


def channel_scores(seed: int, channel: int, frames: int, width: int,
                   dtype=np.float32) -> np.ndarray:
    """Acoustic costs U[0, 6) of one channel from default_rng([seed, channel])
    (random_scores' range, synth.py:69-75; [seed, i] streams, harness.py:374)."""
    x = np.random.default_rng([seed, channel]).uniform(0.0, 6.0, (frames, width))
    return x.astype(dtype) if dtype != np.float64 else x


def unigram_context(csr, num_words: int, ctx_seed: int, *, num_labels: int,
                    discount: float = -2.0, ctx_id: str | None = None) -> BiasingContext:
    """Context of single-word entities: exactly the arcs whose olabel is one of
    the chosen words (single-word completeness of Alg. 1)."""
    words = random.Random(ctx_seed).sample(range(1, num_labels + 1), num_words)
    idx = np.flatnonzero(np.isin(np.asarray(csr.olabels), np.asarray(words)))
    return BiasingContext(id=ctx_id or f"ctx{ctx_seed}", arc_indices=idx.astype(np.int64),
                          discount=discount)


class OlabelIndex:
    """Arcs grouped by output label (one argsort of the olabel array), so the
    unigram contexts of a 2e7-arc graph are built without rescanning it."""

    def __init__(self, csr):
        ol = np.asarray(csr.olabels)
        self.order = np.argsort(ol, kind="stable").astype(np.int64)
        self.sorted = ol[self.order]

    def arcs_of(self, words) -> np.ndarray:
        w = np.asarray(sorted(words))
        lo = np.searchsorted(self.sorted, w, side="left")
        hi = np.searchsorted(self.sorted, w, side="right")
        parts = [self.order[a:b] for a, b in zip(lo, hi)]
        return np.sort(np.concatenate(parts)) if parts else np.zeros(0, dtype=np.int64)


def unigram_contexts(csr, num_words: int, ctx_seeds, *, num_labels: int,
                     discount: float = -2.0) -> list:
    """unigram_context for many seeds sharing one OlabelIndex."""
    ix = OlabelIndex(csr)
    out = []
    for s in ctx_seeds:
        words = random.Random(s).sample(range(1, num_labels + 1), num_words)
        out.append(BiasingContext(id=f"ctx{s}", arc_indices=ix.arcs_of(words), discount=discount))
    return out


def dense_context(csr, fraction: float, ctx_seed: int, *, discount: float = -2.0,
                  ctx_id: str | None = None) -> BiasingContext:
    """Context boosting a uniform random ``fraction`` of all arcs (ATC-style)."""
    rng = np.random.default_rng([ctx_seed, 77])
    n = csr.num_arcs if hasattr(csr, "num_arcs") else int(csr.row_offsets[-1])
    k = int(round(fraction * n))
    idx = np.sort(rng.choice(n, size=k, replace=False)).astype(np.int64)
    return BiasingContext(id=ctx_id or f"dense{ctx_seed}", arc_indices=idx, discount=discount)


def graph_entities(csr, n: int, seed: int, *, min_words: int = 2, max_words: int = 3) -> list:
    """n multi-word entities that occur in the graph: random arc walks that
    output a word at every step (so Alg. 1 has chains to follow and boosts
    more than the first word's arcs, biasing.py:203-233)."""
    rng = random.Random(seed)
    ro, ol, ns = np.asarray(csr.row_offsets), np.asarray(csr.olabels), np.asarray(csr.next_states)
    out = []
    while len(out) < n:
        g = rng.randrange(len(ol))
        words = []
        for _ in range(rng.randint(min_words, max_words)):
            if ol[g] == 0:
                break
            words.append(int(ol[g]))
            s = int(ns[g])
            if ro[s + 1] == ro[s]:
                break
            g = rng.randrange(int(ro[s]), int(ro[s + 1]))
        if len(words) >= min_words:
            out.append(words)
    return out


def entity_contexts(csr, per_context: int, ctx_seeds, *, discount: float = -2.0,
                    depth: int = 10) -> list:
    """Contexts of multi-word entities compiled by the native Alg. 1
    (compiler._compile, all host threads): the C3 contexts of an ATC-style
    deployment (callsigns), not label-closed, so LIST or BITSET on the device."""
    from . import compiler as K

    arrays = K.csr_arrays(csr)
    out = []
    for s in ctx_seeds:
        arcs, _ = K._compile(arrays, graph_entities(csr, per_context, s), depth)
        out.append(BiasingContext(id=f"ent{s}", arc_indices=np.asarray(arcs, dtype=np.int64),
                                  discount=discount))
    return out


def pcg64_streams(seeds) -> np.ndarray:
    """[n, 4] uint64 {state hi, state lo, inc hi, inc lo} of
    ``np.random.default_rng(seed)`` for each seed (numpy's PCG64 state)."""
    out = np.zeros((len(seeds), 4), dtype=np.uint64)
    m = (1 << 64) - 1
    for i, seed in enumerate(seeds):
        st = np.random.default_rng(seed).bit_generator.state["state"]
        s, inc = int(st["state"]), int(st["inc"])
        out[i] = (s >> 64, s & m, inc >> 64, inc & m)
    return out


def device_uniform(seeds, n: int, low: float, high: float, *, offset: float = 0.0,
                   dtype="float32", out=None, device: int = 0):
    """``offset + default_rng(seed).uniform(low, high, n)`` for every seed,
    generated on the GPU bit-identically to numpy (``ab_scores_generate``):
    a [len(seeds), n] torch tensor in device memory."""
    import ctypes as C

    import torch

    from . import _lib

    tdt = torch.float32 if str(dtype) in ("float32", "torch.float32") else torch.float64
    if out is None:
        out = torch.empty((len(seeds), n), dtype=tdt, device=torch.device("cuda", device))
    if not (out.is_cuda and out.is_contiguous() and out.dtype == tdt and out.numel() == len(seeds) * n):
        raise ValueError("out must be a contiguous CUDA tensor of len(seeds) * n values")
    st = np.ascontiguousarray(pcg64_streams(seeds))
    stream = torch.cuda.current_stream(out.device).cuda_stream
    _lib.check(_lib.load().ab_scores_generate(
        out.device.index, st.ctypes.data, len(seeds), int(n), float(low), float(high), float(offset),
        _lib.AB_F32 if tdt == torch.float32 else _lib.AB_F64, C.c_void_p(out.data_ptr()),
        C.c_void_p(stream)))
    return out


def device_channel_scores(seed: int, channels, frames: int, width: int, *, out=None, device: int = 0):
    """``channel_scores(seed, c, frames, width)`` for every c in channels,
    stacked [C, frames, width] f32, generated in device memory."""
    chans = list(channels)
    t = device_uniform([[seed, c] for c in chans], frames * width, 0.0, 6.0,
                       out=None if out is None else out.view(len(chans), frames * width), device=device)
    return t.view(len(chans), frames, width)
