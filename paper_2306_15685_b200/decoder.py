"""Reference-compatible decode API backed by the sm_100a kernels.

Names, argument meaning and error behaviour follow the reference
(/root/reference/pkg/src/arcboost/decoder.py): ``init_channel`` (162-174),
``switch_context`` (177-193), ``advance_frame`` (341-411),
``partial_hypothesis`` (414-423), ``finalize`` (426-460), ``detect_endpoint``
(463-464), ``decode_batch`` (504-526).  A ``Channel`` is a host mirror of a
device channel slot: lifecycle checks that the reference performs before
touching state run on the host; everything that touches tokens runs in the
CUDA library.  There is no CPU decode path: without the library the first
device call raises.

Additions (not in the reference): ``Hypothesis.hits`` is the number of boosted
arcs on the hypothesis path (north-star "boosted-arc hits"; excluded from
equality so hypotheses compare like the reference's).
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass, field
from enum import Enum
from typing import Sequence

import numpy as np

from . import _lib
from .biasing import BiasingContext, ContextRegistry
from .device import BatchDecoder, DeviceGraph, device_graph
from .scores import ScoreMatrix


class DecodeError(RuntimeError):
    """Decoding cannot proceed (dead channel, bad inputs, state misuse)."""


@dataclass(frozen=True)
class DecoderConfig:
    beam: float = 16.0
    max_active: int = 7000
    max_epsilon_expansion: int = 20
    partial_every: int = 10
    endpoint_silence_frames: int = 20
    silence_ilabel: int = 0
    # Not in the reference (decoder.py:33-48).  False: candidates that provably
    # cannot survive the frame are dropped at expansion (same surviving tokens,
    # costs and hypotheses; len(store) and eps_truncations then count the
    # relaxed candidates only).  True: every candidate is relaxed, as the
    # reference does, so those two counters match it too.
    exact_counters: bool = False

    def __post_init__(self) -> None:
        if self.beam <= 0:
            raise ValueError("beam must be positive")
        if self.max_active < 1:
            raise ValueError("max_active must be >= 1")
        if self.partial_every < 1:
            raise ValueError("partial_every must be >= 1")


class ChannelStatus(str, Enum):
    IDLE = "idle"
    DECODING = "decoding"
    ENDPOINTED = "endpointed"
    FINISHED = "finished"


_STATUS_TO_CODE = {ChannelStatus.IDLE: _lib.AB_IDLE, ChannelStatus.DECODING: _lib.AB_DECODING,
                   ChannelStatus.ENDPOINTED: _lib.AB_ENDPOINTED,
                   ChannelStatus.FINISHED: _lib.AB_FINISHED}
_CODE_TO_STATUS = {v: k for k, v in _STATUS_TO_CODE.items()}


@dataclass
class Token:
    """decoder.py:58-62 (state, cost, backpointer).  ``backpointer`` is the
    device emission-record id of the token's newest word (-1 = none); record
    ids are the device arena's, not the reference store's positions (the words
    they lead to are the same).  ``hits`` (boosted arcs on the path) is extra."""
    state: int
    cost: float
    backpointer: int = -1
    hits: int = 0


@dataclass
class Hypothesis:
    words: list
    cost: float
    frame: int
    kind: str
    fallback: bool = False
    hits: int = field(default=0, compare=False)


class _StoreView:
    """len(ch.store) = emission records of the current utterance (decoder.py:82-83)."""

    def __init__(self, ch: "Channel"):
        self._ch = ch

    def __len__(self) -> int:
        return self._ch._store_len


@dataclass
class Channel:
    id: str
    context_id: str | None = None
    status: ChannelStatus = ChannelStatus.IDLE
    frame_index: int = 0
    total_frames: int = 0
    utterance_index: int = 0
    trailing_silence: int = 0
    eps_truncations: int = 0
    _fresh: bool = field(default=True, repr=False)
    _num_active: int = field(default=0, repr=False, compare=False)
    _store_len: int = field(default=0, repr=False, compare=False)
    _graph: DeviceGraph | None = field(default=None, repr=False, compare=False)
    _page: BatchDecoder | None = field(default=None, repr=False, compare=False)
    _slot: int = field(default=-1, repr=False, compare=False)
    _ctx_handle: int = field(default=-1, repr=False, compare=False)
    _last_words: list = field(default_factory=list, repr=False, compare=False)
    _work: tuple = field(default=(0, 0, 0), repr=False, compare=False)
    _slot_finalizer: object = field(default=None, repr=False, compare=False)

    @property
    def store(self) -> _StoreView:
        return _StoreView(self)

    @property
    def num_active(self) -> int:
        return self._num_active

    def active_tokens(self) -> list[Token]:
        if self._page is None or self._num_active == 0:
            return []
        st, co, hi, bp = self._page.tokens(self._slot)
        order = np.lexsort((co, st))
        return [Token(int(st[i]), float(co[i]), int(bp[i]), int(hi[i])) for i in order]

    @property
    def work_counters(self) -> tuple:
        """(token expansions, emitting arcs, epsilon arcs) accumulated on the device."""
        return self._work


# ------------------------------------------------------------ host mirror sync

def _bind(ch: Channel, csr, prefer: BatchDecoder | None = None) -> tuple[BatchDecoder, int]:
    dg = device_graph(csr)
    if ch._graph is dg:
        return ch._page, ch._slot
    if ch._graph is not None:
        if not ch._fresh:
            raise DecodeError(f"channel {ch.id!r}: cannot move to another graph mid-utterance")
        # the old slot goes back now; its finalizer must not free it again later
        # (another channel may own it by then)
        if ch._slot_finalizer is not None:
            ch._slot_finalizer()
    page, slot = dg.bind_slot(prefer)
    ch._graph, ch._page, ch._slot = dg, page, slot
    ch._last_words = []
    ch._slot_finalizer = weakref.finalize(ch, page.free_slot, slot)
    return page, slot


def _push(ch: Channel) -> None:
    info = _lib.ab_channel_info()
    info.status = _STATUS_TO_CODE[ch.status]
    info.fresh = 1 if ch._fresh else 0
    info.frame_index = ch.frame_index
    info.total_frames = ch.total_frames
    info.utterance_index = ch.utterance_index
    info.trailing_silence = ch.trailing_silence
    info.eps_truncations = ch.eps_truncations
    info.context = ch._ctx_handle
    info.num_active = ch._num_active
    info.store_len = ch._store_len
    info.error = 0
    info.tok_expansions, info.emit_arcs, info.eps_arcs = ch._work
    ch._page.put(ch._slot, info)


def _pull(ch: Channel) -> None:
    info = ch._page.get(ch._slot)
    ch.status = _CODE_TO_STATUS[info.status]
    ch._fresh = bool(info.fresh)
    ch.frame_index = info.frame_index
    ch.total_frames = info.total_frames
    ch.utterance_index = info.utterance_index
    ch.trailing_silence = info.trailing_silence
    ch.eps_truncations = info.eps_truncations
    ch._num_active = info.num_active
    ch._store_len = info.store_len
    ch._work = (info.tok_expansions, info.emit_arcs, info.eps_arcs)


def hyp_from_device(h, words: np.ndarray, prev: list) -> tuple[Hypothesis, list]:
    """A device hypothesis row -> Hypothesis.  The device shares path prefixes:
    ``h.shared`` leading words equal the previous hypothesis of the same channel
    (``prev``); the rest are at ``words[h.words_off:]``.  Returns the hypothesis
    and the prefix the channel's next row refers to (empty after a final)."""
    s, n = h.shared, h.n_words
    suffix = words[h.words_off:h.words_off + (n - s)].tolist() if n > s else []
    w = prev[:s] + suffix
    kind = "final" if h.kind == _lib.AB_FINAL else "partial"
    return (Hypothesis(words=list(w), cost=float(h.cost), frame=int(h.frame), kind=kind,
                       fallback=bool(h.fallback), hits=int(h.hits)),
            [] if kind == "final" else w)


def _hyp(ch: Channel, h, words: np.ndarray) -> Hypothesis:
    hyp, ch._last_words = hyp_from_device(h, words, ch._last_words)
    return hyp


def device_error(channel_id: str, status: str, code: int, what: str = "finalize") -> DecodeError:
    """The reference's DecodeError for a device error code (decoder.py:422, 437-441, 459)."""
    if code == _lib.AB_ERR_DEAD:
        return DecodeError(f"channel {channel_id!r}: decode failure, no active tokens")
    if code == _lib.AB_ERR_STATUS:
        return DecodeError(f"channel {channel_id!r}: cannot {what} in status {status}")
    if code == _lib.AB_ERR_CAPACITY:
        return DecodeError(
            f"channel {channel_id!r}: device capacity exceeded (token table, frontier log, emission "
            "arena or hypothesis path); raise paper_2306_15685_b200.device.DEFAULT_CAPACITY")
    return DecodeError(f"channel {channel_id!r}: device error {code}")


def _device_error(ch: Channel, code: int, what: str = "finalize") -> DecodeError:
    return device_error(ch.id, ch.status.value, code, what)


def _width_error(width, L) -> DecodeError:
    return DecodeError(
        f"frame width {width} does not match the graph's emitting-label count {L}")


def _check_eps_cap(cfg) -> None:
    """Any integer cap is accepted, as in the reference (decoder.py:263); the
    device field is int32, so larger caps saturate (same rounds: a closure
    ends long before 2**31 rounds, every round with applications takes a
    frontier row)."""
    int(cfg.max_epsilon_expansion)


# ------------------------------------------------------------------- public API

def init_channel(id: str, registry: ContextRegistry | None, context_id: str | None,
                 cfg: DecoderConfig) -> Channel:
    """decoder.py:162-174: an idle channel; its context must be registered."""
    if context_id is not None:
        if registry is None:
            raise DecodeError("context requested but no registry given")
        registry.get(context_id)
    return Channel(id=id, context_id=context_id)


def switch_context(ch: Channel, registry: ContextRegistry | None,
                   context_id: str | None) -> Channel:
    """decoder.py:177-193: swap the context at an utterance boundary."""
    if ch.status not in (ChannelStatus.IDLE, ChannelStatus.FINISHED):
        raise DecodeError(
            f"channel {ch.id!r}: context switch mid-utterance (status {ch.status.value})")
    if context_id is not None:
        if registry is None:
            raise DecodeError("context requested but no registry given")
        registry.get(context_id)
    ch.context_id = context_id
    if ch.status is ChannelStatus.FINISHED:
        ch.status = ChannelStatus.IDLE
    return ch


def advance_frame(ch: Channel, frame, csr, ctx: BiasingContext | None,
                  cfg: DecoderConfig) -> Channel:
    """decoder.py:341-411: one frame for one channel, on the device."""
    if ch.status not in (ChannelStatus.IDLE, ChannelStatus.DECODING):
        raise DecodeError(f"channel {ch.id!r}: cannot advance in status {ch.status.value}")
    row = np.asarray(frame)
    if row.dtype != np.float32:
        row = np.asarray(row, dtype=np.float64)
    dg = device_graph(csr)
    if row.ndim != 1 or len(row) != dg.num_emitting_labels:
        raise _width_error(row.shape, dg.num_emitting_labels)
    _check_eps_cap(cfg)
    page, slot = _bind(ch, csr)
    ch._ctx_handle = dg.context_handle(ctx)
    _push(ch)
    page.decode([slot], [1], [0], np.ascontiguousarray(row[None, :]), dg.num_emitting_labels, cfg,
                _lib.AB_MODE_ADVANCE)
    nh, er, _, _, _ = page.results(1)
    _pull(ch)
    if er[0]:
        raise _device_error(ch, int(er[0]), "advance")
    return ch


def partial_hypothesis(ch: Channel) -> Hypothesis:
    """decoder.py:414-423."""
    if ch._fresh:
        return Hypothesis(words=[], cost=0.0, frame=ch.total_frames, kind="partial")
    if ch._page is None or ch._num_active == 0:
        raise DecodeError(f"channel {ch.id!r}: decode failure, no active tokens")
    _push(ch)
    rc, h, words = ch._page.one_hyp(ch._slot, final=False)
    if rc != _lib.AB_OK:
        _pull(ch)
        raise _device_error(ch, rc, "partial")
    _pull(ch)
    words_off0 = h.words_off
    h.words_off = 0
    out = _hyp(ch, h, words)
    h.words_off = words_off0
    return out


def finalize(ch: Channel, csr) -> Hypothesis:
    """decoder.py:426-460: best final token (fallback: best token); resets the channel."""
    if ch.status not in (ChannelStatus.DECODING, ChannelStatus.ENDPOINTED) and not (
        ch.status is ChannelStatus.IDLE and ch._fresh
    ):
        raise DecodeError(f"channel {ch.id!r}: cannot finalize in status {ch.status.value}")
    if not ch._fresh and ch._num_active == 0:
        raise DecodeError(f"channel {ch.id!r}: decode failure, no active tokens")
    _bind(ch, csr)
    _push(ch)
    rc, h, words = ch._page.one_hyp(ch._slot, final=True)
    _pull(ch)
    if rc != _lib.AB_OK:
        raise _device_error(ch, rc)
    h.words_off = 0
    return _hyp(ch, h, words)


def detect_endpoint(ch: Channel, cfg: DecoderConfig) -> bool:
    return ch.trailing_silence >= cfg.endpoint_silence_frames


@dataclass
class ChannelResult:
    channel_id: str
    hypotheses: list
    error: str | None = None


def _prepare(ch: Channel, scores: ScoreMatrix, csr, registry, dg: DeviceGraph):
    """The checks _decode_one performs before touching tokens (decoder.py:481-489)."""
    ctx = registry.resolve(ch.context_id) if registry is not None else None
    if ch.context_id is not None and registry is None:
        raise DecodeError(f"channel {ch.id!r} has a context but no registry was given")
    if ctx is not None and registry.graph_fingerprint and \
            registry.graph_fingerprint != csr.fingerprint:
        raise DecodeError(
            f"channel {ch.id!r}: context registry was compiled against a different graph")
    if ch.status is ChannelStatus.FINISHED:
        ch.status = ChannelStatus.IDLE
    T = scores.num_frames
    if T > 0:
        if ch.status not in (ChannelStatus.IDLE, ChannelStatus.DECODING):
            raise DecodeError(f"channel {ch.id!r}: cannot advance in status {ch.status.value}")
        if scores.num_ilabels != dg.num_emitting_labels:
            raise _width_error((scores.num_ilabels,), dg.num_emitting_labels)
    else:
        if ch.status not in (ChannelStatus.DECODING, ChannelStatus.ENDPOINTED) and not (
            ch.status is ChannelStatus.IDLE and ch._fresh
        ):
            raise DecodeError(f"channel {ch.id!r}: cannot finalize in status {ch.status.value}")
    return ctx


def decode_batch(channels: Sequence[tuple[Channel, ScoreMatrix]], csr,
                 registry: ContextRegistry | None, cfg: DecoderConfig,
                 num_workers: int = 1) -> list[ChannelResult]:
    """decoder.py:504-526: every channel's stream decoded in one device launch
    per decoder page (channels are CTAs of the same kernel).  Results keep the
    input order; per-channel errors do not abort the batch.  ``num_workers`` is
    accepted for API compatibility; the device runs all channels at once."""
    results: list[ChannelResult | None] = [None] * len(channels)
    if not channels:
        return []
    dg = device_graph(csr)
    _check_eps_cap(cfg)
    pending: list[tuple[int, Channel, ScoreMatrix]] = []
    page = dg.reserve(len({id(ch) for ch, _ in channels if ch._graph is not dg}))
    for i, (ch, scores) in enumerate(channels):
        try:
            ctx = _prepare(ch, scores, csr, registry, dg)
            _bind(ch, csr, page)
            ch._ctx_handle = dg.context_handle(ctx)
            pending.append((i, ch, scores))
        except Exception as exc:  # per-channel isolation (decoder.py:516-521)
            results[i] = ChannelResult(ch.id, [], error=f"{type(exc).__name__}: {exc}")
    # a channel listed twice decodes its streams in order: split into waves
    while pending:
        wave, rest, seen = [], [], set()
        for item in pending:
            (wave if id(item[1]) not in seen and not seen.add(id(item[1])) else rest).append(item)
        by_page: dict[int, list] = {}
        for item in wave:
            by_page.setdefault(id(item[1]._page), []).append(item)
        for items in by_page.values():
            _launch_stream(items, dg, cfg, results)
        pending = rest
    return results  # type: ignore[return-value]


def pack_streams(mats, L: int) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Score matrices of one launch -> (packed rows, frames per stream, row
    offsets).  f32 when every cost is exactly an f32 (half the H2D bytes, same
    f64 arithmetic on the device), else f64."""
    m32 = []
    f32 = True
    for m in mats:
        if f32:
            x = m if m.dtype == np.float32 else m.astype(np.float32)
            f32 = x is m or np.array_equal(x, m)
            m32.append(x)
    src = m32 if f32 else [m.astype(np.float64, copy=False) for m in mats]
    frames = np.array([m.shape[0] for m in mats], dtype=np.int32)
    offs = np.zeros(len(mats), dtype=np.int64)
    if len(mats) > 1:
        np.cumsum(frames[:-1].astype(np.int64) * L, out=offs[1:])
    rows = [m.reshape(-1) for m in src if m.size]
    dt = np.float32 if f32 else np.float64
    packed = np.ascontiguousarray(np.concatenate(rows)) if rows else np.zeros(1, dtype=dt)
    return packed, frames, offs


def _launch_stream(items, dg: DeviceGraph, cfg, results) -> None:
    page = items[0][1]._page
    L = dg.num_emitting_labels
    packed, frames, offs = pack_streams([s.costs for _, _, s in items], L)
    for _, ch, _ in items:
        _push(ch)
    page.decode([ch._slot for _, ch, _ in items], frames, offs, packed, L, cfg,
                _lib.AB_MODE_STREAM)
    nh, er, hyps, stride, words = page.results(len(items))
    for j, (i, ch, _) in enumerate(items):
        hs = [_hyp(ch, hyps[j * stride + q], words) for q in range(int(nh[j]))]
        _pull(ch)
        if er[j]:
            results[i] = ChannelResult(ch.id, [], error=f"DecodeError: {_device_error(ch, int(er[j]))}")
        else:
            results[i] = ChannelResult(ch.id, hs)
