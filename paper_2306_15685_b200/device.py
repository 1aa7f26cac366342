"""Device resources behind the reference-compatible API.

``DeviceGraph`` owns one uploaded graph (``ab_graph``) and its context store;
``BatchDecoder`` owns the per-channel device pools of up to ``max_channels``
channels (``ab_decoder``).  The reference API (decoder.py) binds each
``Channel`` lazily to a slot of a decoder page of the graph it is decoded on.
Everything here calls the CUDA library; nothing runs on the CPU.
"""

from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def default_device() -> int:
    """The GPU a graph goes to when the caller names none.  In order:
    ``ARCBOOST_DEVICE``; torch's current device when torch has initialised
    CUDA in this process (a rank that called ``torch.cuda.set_device``);
    ``LOCAL_RANK`` modulo the device count (one process per GPU under
    torchrun); else 0."""
    env = os.environ.get("ARCBOOST_DEVICE")
    if env is not None:
        return int(env)
    import sys

    torch = sys.modules.get("torch")
    if torch is not None:
        try:
            if torch.cuda.is_initialized():
                return int(torch.cuda.current_device())
        except Exception:
            pass
    local = os.environ.get("LOCAL_RANK")
    if local is not None:
        n = C.c_int32()
        if _lib.load().ab_device_count(C.byref(n)) == 0 and n.value > 0:
            return int(local) % n.value
    return 0


class DeviceGraph:
    """Device CSR split into emitting / epsilon SoA (fst.py:165-191)."""

    def __init__(self, csr, device: int | None = None):
        lib = _lib.load()
        if device is None:
            device = default_device()
        self.device = device
        ro = np.ascontiguousarray(csr.row_offsets, dtype=np.int64)
        il = np.ascontiguousarray(csr.ilabels, dtype=np.int32)
        ol = np.ascontiguousarray(csr.olabels, dtype=np.int32)
        ns = np.ascontiguousarray(csr.next_states, dtype=np.int32)
        w = np.ascontiguousarray(csr.weights, dtype=np.float64)
        finals = csr.finals
        if hasattr(finals, "as_arrays"):
            fs, fc = finals.as_arrays()
            fs = np.ascontiguousarray(fs, dtype=np.int32)
            fc = np.ascontiguousarray(fc, dtype=np.float64)
        elif isinstance(finals, dict):
            fs = np.fromiter(finals.keys(), dtype=np.int32, count=len(finals))
            fc = np.fromiter(finals.values(), dtype=np.float64, count=len(finals))
        else:  # (states, costs) arrays
            fs = np.ascontiguousarray(finals[0], dtype=np.int32)
            fc = np.ascontiguousarray(finals[1], dtype=np.float64)
        self.num_states = len(ro) - 1
        self.num_arcs = int(ro[-1]) if len(ro) else 0
        h = C.c_void_p()
        check(lib.ab_graph_create(device, int(csr.start), self.num_states, self.num_arcs,
                                  _ptr(ro), _ptr(il), _ptr(ol), _ptr(ns), _ptr(w), len(fs),
                                  _ptr(fs), _ptr(fc), C.byref(h)))
        self.handle = h.value
        L = C.c_int32()
        w32 = C.c_int32()
        nbytes = C.c_int64()
        check(lib.ab_graph_query(self.handle, C.byref(L), C.byref(w32), C.byref(nbytes)))
        self.num_emitting_labels = L.value
        self.weights_f32 = bool(w32.value)
        self.device_bytes = nbytes.value
        self._ctx: dict[int, tuple[weakref.ref, int, tuple]] = {}
        self._pages: list[BatchDecoder] = []
        # decoders built on this graph must be destroyed before it
        self._decoder_finalizers: list = []
        self._finalizer = weakref.finalize(self, _destroy_graph, self.handle,
                                           self._decoder_finalizers)

    # -- context store -------------------------------------------------
    def register_context(self, arc_indices, discount: float, mode: int = _lib.AB_CTX_AUTO) -> int:
        idx = np.ascontiguousarray(arc_indices, dtype=np.int64)
        h = C.c_int32()
        check(_lib.load().ab_context_register(self.handle, _ptr(idx), len(idx), float(discount),
                                              int(mode), C.byref(h)))
        return h.value

    def context_mode(self, handle: int) -> int:
        m = C.c_int32()
        check(_lib.load().ab_context_mode(self.handle, int(handle), C.byref(m)))
        return m.value

    def context_slack(self, handle: int) -> tuple[float, int]:
        """(epsilon slack, set bits of its Bloom filter of slack states) of a
        context (-1: unbiased); the count is negative when the slack bounds
        paths of at most 64 epsilon arcs only (ab_context_slack)."""
        v = C.c_double()
        n = C.c_int32()
        check(_lib.load().ab_context_slack(self.handle, int(handle), C.byref(v), C.byref(n)))
        return v.value, n.value

    def release_context(self, handle: int) -> None:
        check(_lib.load().ab_context_release(self.handle, int(handle)))

    def context_handle(self, ctx) -> int:
        """Device handle of a BiasingContext (registered on first use)."""
        if ctx is None:
            return -1
        key = id(ctx)
        # the reference reads the live object every frame (decoder.py:234-240):
        # a changed discount or a reassigned index array is a new device context
        arcs = ctx.arc_indices
        n = len(arcs)
        stamp = (float(ctx.discount), id(arcs), n, int(arcs[0]) if n else -1, int(arcs[-1]) if n else -1)
        hit = self._ctx.get(key)
        if hit is not None and hit[0]() is ctx and hit[2] == stamp:
            return hit[1]
        h = self.register_context(arcs, ctx.discount)
        self._ctx[key] = (weakref.ref(ctx, lambda _r, k=key, hh=h: self._drop_ctx(k, hh)), h, stamp)
        return h

    def _drop_ctx(self, key: int, h: int) -> None:
        cur = self._ctx.get(key)
        if cur is not None and cur[1] == h:
            del self._ctx[key]
            try:
                self.release_context(h)
            except Exception:
                pass

    # -- channel slots -------------------------------------------------
    def reserve(self, n: int) -> "BatchDecoder | None":
        """A page with room for n more channels (a new one if none has it), so
        a batch binding many channels at once decodes in one launch instead of
        one per geometrically grown page."""
        if n <= 0:
            return None
        for p in self._pages:
            if len(p._free) >= n:
                return p
        p = BatchDecoder(self, min(1024, max(n, 8 << len(self._pages))))
        self._pages.append(p)
        return p

    def bind_slot(self, prefer: "BatchDecoder | None" = None) -> tuple["BatchDecoder", int]:
        if prefer is not None:
            s = prefer.alloc_slot()
            if s is not None:
                return prefer, s
        for p in self._pages:
            s = p.alloc_slot()
            if s is not None:
                return p, s
        size = min(1024, 8 << len(self._pages))
        p = BatchDecoder(self, size)
        self._pages.append(p)
        return p, p.alloc_slot()


def _destroy_graph(handle, decoder_finalizers):
    for f in decoder_finalizers:
        f()
    try:
        _lib.load().ab_graph_destroy(handle)
    except Exception:
        pass


def _destroy_decoder(handle):
    try:
        _lib.load().ab_decoder_destroy(handle)
    except Exception:
        pass


@dataclass
class Capacity:
    table_slots: int = 0
    frontier_rows: int = 0
    arena_records: int = 0
    path_words: int = 0


DEFAULT_CAPACITY = Capacity()


class BatchDecoder:
    """Per-channel device pools for up to ``max_channels`` channels of one graph."""

    def __init__(self, graph: DeviceGraph, max_channels: int, capacity: Capacity | None = None):
        cap = capacity or DEFAULT_CAPACITY
        c = _lib.ab_capacity(cap.table_slots, cap.frontier_rows, cap.arena_records,
                             cap.path_words)
        h = C.c_void_p()
        check(_lib.load().ab_decoder_create(graph.handle, C.byref(c), int(max_channels),
                                            C.byref(h)))
        self.graph = graph
        self.handle = h.value
        self.max_channels = max_channels
        self._free = list(range(max_channels - 1, -1, -1))
        q = _lib.ab_capacity()
        nb = C.c_int64()
        check(_lib.load().ab_decoder_query(self.handle, C.byref(q), C.byref(nb)))
        self.capacity = Capacity(q.table_slots, q.frontier_rows, q.arena_records, q.path_words)
        self.device_bytes = nb.value
        self._finalizer = weakref.finalize(self, _destroy_decoder, self.handle)
        graph._decoder_finalizers.append(self._finalizer)

    def alloc_slot(self) -> int | None:
        if not self._free:
            return None
        s = self._free.pop()
        self.init_channel(s, -1)
        return s

    def free_slot(self, s: int) -> None:
        self._free.append(s)

    def init_channel(self, slot: int, ctx: int = -1) -> None:
        check(_lib.load().ab_channel_init(self.handle, int(slot), int(ctx)))

    def get(self, slot: int) -> _lib.ab_channel_info:
        info = _lib.ab_channel_info()
        check(_lib.load().ab_channel_get(self.handle, int(slot), C.byref(info)))
        return info

    def put(self, slot: int, info: _lib.ab_channel_info) -> None:
        check(_lib.load().ab_channel_put(self.handle, int(slot), C.byref(info)))

    def tokens(self, slot: int):
        n = C.c_int32()
        check(_lib.load().ab_channel_tokens(self.handle, int(slot), None, None, None, None, 0,
                                            C.byref(n)))
        st = np.zeros(max(n.value, 1), dtype=np.int32)
        co = np.zeros(max(n.value, 1), dtype=np.float64)
        hi = np.zeros(max(n.value, 1), dtype=np.int32)
        bp = np.zeros(max(n.value, 1), dtype=np.int32)
        check(_lib.load().ab_channel_tokens(self.handle, int(slot), _ptr(st), _ptr(co), _ptr(hi),
                                            _ptr(bp), n.value, C.byref(n)))
        return st[:n.value], co[:n.value], hi[:n.value], bp[:n.value]

    def decode(self, slots, frames, score_offsets, scores, width: int, cfg, mode: int,
               scores_on_device: bool = False, scores_dtype: int | None = None,
               stream: int | None = None) -> None:
        """Launch one batch (decode_batch / advance_frame × T); results stay queued."""
        slots = np.ascontiguousarray(slots, dtype=np.int32)
        frames = np.ascontiguousarray(frames, dtype=np.int32)
        offs = np.ascontiguousarray(score_offsets, dtype=np.int64)
        a = _lib.ab_decode_args()
        a.n = len(slots)
        a.channels = _ptr(slots)
        a.frames = _ptr(frames)
        a.score_offsets = _ptr(offs)
        if scores_on_device:
            a.scores = int(scores)
            a.scores_dtype = int(scores_dtype)
        else:
            a.scores = _ptr(scores) if scores is not None and scores.size else None
            a.scores_dtype = _lib.AB_F32 if (scores is not None and scores.dtype == np.float32) \
                else _lib.AB_F64
        a.scores_on_device = 1 if scores_on_device else 0
        a.width = int(width)
        a.mode = int(mode)
        a.config = make_config(cfg)
        a.stream = stream
        check(_lib.load().ab_decode(self.handle, C.byref(a)))

    def results(self, n: int):
        """(n_hyps[n], errors[n], hyps[n][...] as ab_hyp rows, words array)."""
        lib = _lib.load()
        nh = np.zeros(max(n, 1), dtype=np.int32)
        er = np.zeros(max(n, 1), dtype=np.int32)
        used = C.c_int64()
        check(lib.ab_read_results(self.handle, _ptr(nh), _ptr(er), None, 0, None, 0,
                                  C.byref(used)))
        stride = int(nh[:n].max()) if n else 0
        hyps = (_lib.ab_hyp * max(1, n * stride))()
        words = np.zeros(max(1, used.value), dtype=np.int32)
        check(lib.ab_read_results(self.handle, _ptr(nh), _ptr(er), C.addressof(hyps),
                                  max(stride, 1), _ptr(words), len(words), C.byref(used)))
        return nh[:n], er[:n], hyps, max(stride, 1), words

    def one_hyp(self, slot: int, final: bool):
        lib = _lib.load()
        h = _lib.ab_hyp()
        cap = self.capacity.path_words
        words = np.zeros(max(cap, 1), dtype=np.int32)
        fn = lib.ab_finalize if final else lib.ab_partial
        rc = fn(self.handle, int(slot), C.byref(h), _ptr(words), len(words))
        return rc, h, words

    def init_channels(self, slots, contexts) -> None:
        s = np.ascontiguousarray(slots, dtype=np.int32)
        c = np.ascontiguousarray(contexts, dtype=np.int32)
        check(_lib.load().ab_channels_init(self.handle, len(s), _ptr(s), _ptr(c)))

    def set_contexts(self, slots, contexts) -> None:
        """Batched switch_context (decoder.py:177-193) on device slots."""
        s = np.ascontiguousarray(slots, dtype=np.int32)
        c = np.ascontiguousarray(contexts, dtype=np.int32)
        check(_lib.load().ab_channels_set_context(self.handle, len(s), _ptr(s), _ptr(c)))

    def get_many(self, slots) -> list:
        s = np.ascontiguousarray(slots, dtype=np.int32)
        infos = (_lib.ab_channel_info * max(len(s), 1))()
        check(_lib.load().ab_channels_get(self.handle, len(s), _ptr(s), C.addressof(infos)))
        return [infos[i] for i in range(len(s))]

    def last_launch_count(self) -> int:
        n = C.c_int32()
        check(_lib.load().ab_last_launch_count(self.handle, C.byref(n)))
        return n.value

    def last_kernel_ms(self) -> float:
        ms = C.c_float()
        check(_lib.load().ab_last_kernel_ms(self.handle, C.byref(ms)))
        return ms.value


def make_config(cfg) -> _lib.ab_config:
    # the epsilon cap saturates to int32 (same rounds, see decoder._check_eps_cap)
    eps = max(-(1 << 31), min(int(cfg.max_epsilon_expansion), _lib.AB_MAX_EPSILON_ROUNDS))
    flags = _lib.AB_CFG_EXACT if getattr(cfg, "exact_counters", False) else 0
    return _lib.ab_config(float(cfg.beam), int(cfg.max_active), eps,
                          int(cfg.partial_every), int(cfg.endpoint_silence_frames),
                          int(cfg.silence_ilabel), flags)


def device_graph(csr, device: int | None = None) -> DeviceGraph:
    """Cached DeviceGraph of a CsrFst-like object (attribute cache on the object)."""
    dg = getattr(csr, "_ab_device_graph", None)
    if dg is None:
        dg = DeviceGraph(csr, device)
        try:
            object.__setattr__(csr, "_ab_device_graph", dg)
        except Exception:
            pass
    return dg
