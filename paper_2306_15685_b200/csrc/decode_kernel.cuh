// Batched, frame-synchronous, biased token passing on sm_100a.
//
// One CTA owns one channel (a stream) for the whole call and runs every frame
// of it: score-row staging, emitting expansion with the fused boost lookup,
// bounded epsilon closure, beam + max_active pruning, partial / final
// traceback.  Channels are independent, so a launch of n
// CTAs decodes n channels with no inter-CTA synchronisation; with >= ~600
// channels every SM holds several resident channels whose dependent memory
// chains overlap.
//
// Reference semantics reproduced exactly (decoder.py):
//   emitting winner per destination = min (cost, global arc id)        213-220, 367-398
//   epsilon round winner applied iff new state or strictly cheaper     250-316
//   prune: cost <= best + beam, then max_active smallest (cost, state) 319-334
//   best token / partial / final by (cost, state)                     337-338, 414-460
// Costs accumulate in f64 in the reference's association order:
//   emitting (c + w_eff) + score[il-1], epsilon c + w_eff, final c + final[s].
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/arcboost_b200.h"

namespace ab {

typedef unsigned long long u64;
typedef uint32_t u32;

constexpr u64 KEY_PENDING = 1ull << 63;
constexpr u64 KEY_EPOCH_MASK = 0x7FFFFFFF00000000ull;
constexpr u32 SRC_MASK = 0x7FFFFFu;
constexpr int CTX_SMEM_MAX = 1024;          // sparse contexts live in shared memory
constexpr int SCORE_SMEM_MAX_BYTES = 32768; // larger score rows are read from L2

// Token provenance carried with every token (decoder.py:58-62 + last_il 138).
struct __align__(16) TokInfo {
  int bp;      // emission-arena record id, -1 = utterance start
  int depth;   // words on the path (records reachable from bp)
  int hits;    // boosted arcs on the path
  int last_il; // ilabel of the last emitting arc (decoder.py:393, 404)
};

// Token-table slot (32 B = one sector).  key: state | epoch<<32 | PENDING.
// value (16 B, CAS-128 target): ordered cost key, global arc id, info =
// round(8) | boosted(1) | src(23).
struct __align__(32) Entry {
  u64 key;
  u32 flog; // frontier-log row of the latest application
  u32 pad;
  u64 ck;
  u32 g;
  u32 info;
};

struct CtxDesc {
  double discount;
  u32 k;
  int mode; // AB_CTX_LIST / AB_CTX_BITSET
  const u32 *list;
  const u32 *bits;
};

template <typename W> struct EArc;
template <> struct __align__(16) EArc<float> { u32 ns, il, g; float w; };
template <> struct __align__(8) EArc<double> { u32 ns, il, g, pad; double w; };
template <typename W> struct XArc;
template <> struct __align__(16) XArc<float> { u32 ns, g; float w; u32 pad; };
template <> struct __align__(16) XArc<double> { u32 ns, g; double w; };

struct ChanState {
  ab_channel_info info; // info.store_len = records appended this utterance (reference len(store))
  u32 epoch;
  int path_len;
  int max_depth;  // deepest token path in the current token list
  int arena_half; // which half of the channel's arena is live (copying GC)
  u32 rec_phys;   // records physically in the live half
  u32 pad[3];
};

struct DevHyp {
  double cost;
  long long frame;
  int kind, fallback, hits, shared, n_words, pad;
  long long words_off;
};

struct DecodeParams {
  // graph (device CSR split into emitting / epsilon arcs, fst.py:116-191)
  const u32 *e_off;
  const void *e_arcs;
  const u32 *x_off;
  const void *x_arcs;
  const int2 *arc_meta; // [num_arcs] {olabel, ilabel} by global arc id
  const double *final_cost; // NaN = not final
  int start;
  int num_states;
  int L;
  const CtxDesc *ctxs;
  int num_ctxs;
  // per-channel pools (slot-major)
  ChanState *chans;
  Entry *table;
  u32 table_cap, table_mask, hash_shift;
  int hashed;
  u32 *tok_state;
  double *tok_cost;
  TokInfo *tok_info;
  u32 tok_cap;
  u32 *flog_state;
  double *flog_cost;
  TokInfo *flog_info;
  u32 flog_cap;
  u32 *all_list;
  u32 *app_list;
  u64 *scr_key;
  u32 *scr_slot;
  int2 *arena;   // [channel][2][arena_cap]: live half + GC to-space
  u32 arena_cap;
  u32 *gc_bits;  // [channel][arena_cap / 32] mark bitmap
  u32 *gc_rank;  // [channel][arena_cap / 32] live records before each bitmap word
  int *path_rec;
  int *path_words;
  u32 path_cap;
  // batch
  int n;
  const int *slots;
  const int *frames;
  const long long *score_off;
  const void *scores;
  int mode;
  // config (decoder.py:33-48)
  double beam;
  int max_active, max_eps, partial_every, endpoint_silence_frames, silence_ilabel;
  // outputs
  DevHyp *hyps;        // [n, hyp_stride]
  int hyp_stride;
  int *n_hyps;         // [n]
  int *errors;         // [n]
  int *frames_done;    // [n] frames consumed by this launch (pause/resume)
  int *words;          // [n, words_stride] per-channel word regions
  long long words_stride;
  long long *words_used; // [n]
};

// ---------------------------------------------------------------- helpers

__device__ __forceinline__ u64 cost_key(double x) {
  u64 b = (u64)__double_as_longlong(x);
  if (b == 0x8000000000000000ull) b = 0; // -0.0 == +0.0
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_cost(u64 k) {
  u64 b = (k & 0x8000000000000000ull) ? (k & ~0x8000000000000000ull) : ~k;
  return __longlong_as_double((long long)b);
}

__device__ __forceinline__ u64 ld_cg_u64(const u64 *p) {
  u64 v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void ld_cg_value(const Entry *e, u64 &ck, u32 &g, u32 &info) {
  u64 a, b;
  asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(&e->ck));
  ck = a;
  g = (u32)b;
  info = (u32)(b >> 32);
}
__device__ __forceinline__ void st_cg_value(Entry *e, u64 ck, u32 g, u32 info) {
  u64 b = ((u64)info << 32) | g;
  asm volatile("st.global.cg.v2.u64 [%0], {%1, %2};" ::"l"(&e->ck), "l"(ck), "l"(b) : "memory");
}
// 128-bit compare-and-swap on the value half of an entry (ATOMG.E.CAS.128).
__device__ __forceinline__ bool cas_value(Entry *e, u64 &ck, u32 &g, u32 &info, u64 nck, u32 ng,
                                          u32 ninfo) {
  u64 e0 = ck, e1 = ((u64)info << 32) | g;
  u64 d0 = nck, d1 = ((u64)ninfo << 32) | ng;
  u64 r0, r1;
  asm volatile(
      "{\n .reg .b128 e, d, r;\n mov.b128 e, {%2, %3};\n mov.b128 d, {%4, %5};\n"
      " atom.global.cas.b128 r, [%6], e, d;\n mov.b128 {%0, %1}, r;\n}\n"
      : "=l"(r0), "=l"(r1)
      : "l"(e0), "l"(e1), "l"(d0), "l"(d1), "l"(&e->ck)
      : "memory");
  bool ok = (r0 == e0) && (r1 == e1);
  ck = r0;
  g = (u32)r1;
  info = (u32)(r1 >> 32);
  return ok;
}

template <int BLOCK> __device__ __forceinline__ u32 block_excl_scan(u32 v, u32 &total, u32 *sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int NW = BLOCK / 32;
  u32 x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    u32 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    u32 w = lane < NW ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      u32 y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NW) sh[lane] = w;
  }
  __syncthreads();
  u32 base = wid ? sh[wid - 1] : 0;
  total = sh[NW - 1];
  __syncthreads();
  return base + x - v;
}

// (key, state) lexicographic argmin over a block; returns the winner's idx.
template <int BLOCK>
__device__ __forceinline__ void block_argmin(u64 &key, u32 &state, int &idx, u64 *shk, u32 *shs,
                                             int *shi) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int NW = BLOCK / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    u64 k2 = __shfl_xor_sync(0xffffffffu, key, o);
    u32 s2 = __shfl_xor_sync(0xffffffffu, state, o);
    int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    if (k2 < key || (k2 == key && s2 < state)) key = k2, state = s2, idx = i2;
  }
  if (lane == 0) shk[wid] = key, shs[wid] = state, shi[wid] = idx;
  __syncthreads();
  if (wid == 0) {
    key = lane < NW ? shk[lane] : ~0ull;
    state = lane < NW ? shs[lane] : 0xFFFFFFFFu;
    idx = lane < NW ? shi[lane] : -1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      u64 k2 = __shfl_xor_sync(0xffffffffu, key, o);
      u32 s2 = __shfl_xor_sync(0xffffffffu, state, o);
      int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
      if (k2 < key || (k2 == key && s2 < state)) key = k2, state = s2, idx = i2;
    }
    if (lane == 0) shk[0] = key, shs[0] = state, shi[0] = idx;
  }
  __syncthreads();
  key = shk[0];
  state = shs[0];
  idx = shi[0];
  __syncthreads();
}

template <int BLOCK> __device__ __forceinline__ u64 block_min_u64(u64 v, u64 *sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int NW = BLOCK / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = lane < NW ? sh[lane] : ~0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) sh[0] = v;
  }
  __syncthreads();
  v = sh[0];
  __syncthreads();
  return v;
}

// ------------------------------------------------------------ CTA state

enum {
  E_NONE = 0,
  E_DEAD = AB_ERR_DEAD,
  E_STATUS = AB_ERR_STATUS,
  E_CAP = AB_ERR_CAPACITY
};

struct Shared {
  // per-phase counters
  u32 n_all, n_app, n_cand, rec_n, n_keep, n_tok, flog_n;
  unsigned long long rec_logical;
  int error;
  u32 sel;
  u32 cum;
  int shared_words;
  int max_depth;
  long long words_off;
  unsigned long long cnt_tok, cnt_emit, cnt_eps;
  // scan / reduce scratch
  u32 scan[32];
  u64 redk[32];
  u32 reds[32];
  int redi[32];
  u32 hist[256];
};

template <typename W, typename S> struct Chan {
  const DecodeParams *P;
  int slot;
  ChanState *cs;
  Entry *table;
  u32 *tok_state;
  double *tok_cost;
  TokInfo *tok_info;
  u32 *flog_state;
  double *flog_cost;
  TokInfo *flog_info;
  u32 *all_list;
  u32 *app_list;
  u64 *scr_key;
  u32 *scr_slot;
  int2 *arena;   // live half
  int2 *arena_to;
  u32 *gc_bits;
  u32 *gc_rank;
  int *path_rec;
  int *path_words;
  const S *row;
  // context
  double discount;
  int ctx_mode; // 0 none, 1 smem list, 2 global list, 3 bitset
  const u32 *ctx_list;
  u32 ctx_k;
  const u32 *ctx_bits;
  u32 epoch;
};

template <typename W, typename S>
__device__ __forceinline__ bool is_boosted(const Chan<W, S> &C, u32 g) {
  if (C.ctx_mode == 0) return false;
  if (C.ctx_mode == 3) return (__ldg(&C.ctx_bits[g >> 5]) >> (g & 31)) & 1u;
  // BiasingContext.boosted_mask: binary search in the sorted list (biasing.py:108-117)
  const u32 *a = C.ctx_list;
  u32 lo = 0, hi = C.ctx_k;
  while (lo < hi) {
    u32 mid = (lo + hi) >> 1;
    u32 v = a[mid];
    if (v == g) return true;
    if (v < g) lo = mid + 1;
    else hi = mid;
  }
  return false;
}

__device__ __forceinline__ void set_error(Shared &sh, int code) { atomicCAS(&sh.error, 0, code); }

// Relaxation of one candidate into the token table (decoder.py:213-220 for the
// emitting pass; 277-308 for epsilon rounds).  Claims the slot if the state is
// new this epoch; otherwise CAS-128 minimum with the phase rule:
//   value from an earlier round -> replace iff strictly cheaper (cost only)
//   value from this round       -> replace iff (cost, arc) is smaller
template <typename W, typename S>
__device__ __forceinline__ void relax(const Chan<W, S> &C, Shared &sh, u32 d, u64 ck, u32 g,
                                      u32 info, u32 round) {
  const DecodeParams &P = *C.P;
  u32 slot = P.hashed ? ((d * 2654435761u) >> P.hash_shift) & P.table_mask : d;
  const u64 ep = (u64)C.epoch << 32;
  u32 probes = 0;
  while (true) {
    Entry *e = &C.table[slot];
    u64 k = ld_cg_u64(&e->key);
    if ((k & KEY_EPOCH_MASK) != ep) {
      u64 want = (u64)d | ep | KEY_PENDING;
      u64 old = atomicCAS(&e->key, k, want);
      if (old == k) {
        st_cg_value(e, ck, g, info);
        __threadfence();
        atomicExch(&e->key, (u64)d | ep);
        u32 ia = atomicAdd(&sh.n_all, 1u);
        if (ia < P.table_cap) C.all_list[ia] = slot;
        else set_error(sh, E_CAP);
        u32 ip = atomicAdd(&sh.n_app, 1u);
        if (ip < P.table_cap) C.app_list[ip] = slot;
        return;
      }
      continue; // lost the claim race: re-examine the slot
    }
    if ((u32)k != d) {
      slot = (slot + 1) & P.table_mask;
      if (++probes > P.table_mask) {
        set_error(sh, E_CAP);
        return;
      }
      continue;
    }
    while (k & KEY_PENDING) {
      __nanosleep(20);
      k = ld_cg_u64(&e->key);
    }
    __threadfence();
    u64 cck;
    u32 cg, cinfo;
    ld_cg_value(e, cck, cg, cinfo);
    while (true) {
      u32 cround = cinfo >> 24;
      bool better = (cround < round) ? (ck < cck) : (ck < cck || (ck == cck && g < cg));
      if (!better) return;
      if (cas_value(e, cck, cg, cinfo, ck, g, info)) {
        if (cround < round) {
          u32 ip = atomicAdd(&sh.n_app, 1u);
          if (ip < P.table_cap) C.app_list[ip] = slot;
        }
        return;
      }
    }
  }
}

// Load-balanced expansion of a token list over one CSR (emitting or epsilon):
// tiles of BLOCK tokens, block scan of out-degrees, then each thread walks arc
// positions and locates its token by binary search over the tile prefix.
template <int BLOCK, bool EMIT, typename W, typename S>
__device__ void expand(const Chan<W, S> &C, Shared &sh, const u32 *in_state,
                       const double *in_cost, u32 n_in, u32 round) {
  const DecodeParams &P = *C.P;
  __shared__ u32 t_a0[BLOCK];
  __shared__ u32 t_pref[BLOCK];
  __shared__ double t_cost[BLOCK];
  const int tid = threadIdx.x;
  const u32 *off = EMIT ? P.e_off : P.x_off;
  u32 arcs_seen = 0;
  for (u32 base = 0; base < n_in; base += BLOCK) {
    u32 i = base + tid;
    u32 cnt = 0, a0 = 0;
    double c = 0.0;
    if (i < n_in) {
      u32 s = in_state[i];
      c = in_cost[i];
      a0 = __ldg(&off[s]);
      cnt = __ldg(&off[s + 1]) - a0;
    }
    u32 total;
    u32 ex = block_excl_scan<BLOCK>(cnt, total, sh.scan);
    t_a0[tid] = a0;
    t_pref[tid] = ex;
    t_cost[tid] = c;
    __syncthreads();
    arcs_seen += total;
    for (u32 k = tid; k < total; k += BLOCK) {
      // largest j with t_pref[j] <= k (its count is > 0)
      u32 lo = 0, hi = BLOCK - 1;
      while (lo < hi) {
        u32 mid = (lo + hi + 1) >> 1;
        if (t_pref[mid] <= k) lo = mid;
        else hi = mid - 1;
      }
      const u32 j = lo;
      const u32 a = t_a0[j] + (k - t_pref[j]);
      const double cj = t_cost[j];
      u32 ns, g, il = 0;
      double w;
      if (EMIT) {
        const EArc<W> r = reinterpret_cast<const EArc<W> *>(P.e_arcs)[a];
        ns = r.ns;
        il = r.il;
        g = r.g;
        w = (double)r.w;
      } else {
        const XArc<W> r = reinterpret_cast<const XArc<W> *>(P.x_arcs)[a];
        ns = r.ns;
        g = r.g;
        w = (double)r.w;
      }
      // _effective_weights (decoder.py:234-240): boost fused into the cost add
      const bool bst = is_boosted(C, g);
      const double we = bst ? w + C.discount : w;
      double cand;
      if (EMIT) cand = (cj + we) + (double)C.row[il - 1]; // decoder.py:378
      else cand = cj + we;                                 // decoder.py:268
      const u32 info = (round << 24) | (bst ? (1u << 23) : 0u) | ((base + j) & SRC_MASK);
      relax(C, sh, ns, cost_key(cand), g, info, round);
    }
    __syncthreads();
  }
  if (tid == 0) {
    sh.n_cand += arcs_seen;
    sh.cnt_tok += n_in;
    if (EMIT) sh.cnt_emit += arcs_seen;
    else sh.cnt_eps += arcs_seen;
  }
}

// Snapshot of the slots applied in one phase into the frontier log: resolves
// the winner's provenance, appends emission records for olabel != 0
// (decoder.py:385-389, 289-295) and points the slot at its log row.
template <int BLOCK, typename W, typename S>
__device__ void snapshot(const Chan<W, S> &C, Shared &sh, u32 round, const TokInfo *src_info,
                         u32 n_app, u32 row_base) {
  const DecodeParams &P = *C.P;
  if (row_base + n_app > P.flog_cap) {
    if (threadIdx.x == 0) set_error(sh, E_CAP);
    return;
  }
  for (u32 i = threadIdx.x; i < n_app; i += BLOCK) {
    const u32 slot = C.app_list[i];
    Entry *e = &C.table[slot];
    const u32 d = (u32)ld_cg_u64(&e->key);
    u64 ck;
    u32 g, info;
    ld_cg_value(e, ck, g, info);
    const TokInfo si = src_info[info & SRC_MASK];
    const int2 meta = __ldg(&P.arc_meta[g]);
    TokInfo ni;
    ni.bp = si.bp;
    ni.depth = si.depth;
    ni.hits = si.hits + ((info >> 23) & 1);
    ni.last_il = round == 0 ? meta.y : si.last_il;
    if (meta.x != 0) {
      atomicAdd(&sh.rec_logical, 1ull);
      u32 r = atomicAdd(&sh.rec_n, 1u);
      if (r < P.arena_cap) {
        C.arena[r] = make_int2(meta.x, si.bp);
        ni.bp = (int)r;
        ni.depth = si.depth + 1;
      } else {
        set_error(sh, E_CAP);
      }
    }
    const u32 row = row_base + i;
    C.flog_state[row] = d;
    C.flog_cost[row] = key_cost(ck);
    C.flog_info[row] = ni;
    e->flog = row;
  }
}

// _epsilon_rounds (decoder.py:250-316) starting from frontier rows
// [fbase, fbase + nf) of the frontier log.
template <int BLOCK, typename W, typename S>
__device__ void epsilon_rounds(const Chan<W, S> &C, Shared &sh, u32 fbase, u32 nf) {
  const DecodeParams &P = *C.P;
  int rounds = 0;
  while (true) {
    if (!(nf > 0 && rounds < P.max_eps)) {
      if (nf > 0 && threadIdx.x == 0) C.cs->info.eps_truncations += 1; // while-else 314-316
      break;
    }
    rounds++;
    if (threadIdx.x == 0) {
      sh.n_app = 0;
      sh.n_cand = 0;
    }
    __syncthreads();
    expand<BLOCK, false>(C, sh, C.flog_state + fbase, C.flog_cost + fbase, nf, (u32)rounds);
    __syncthreads();
    const u32 n_cand = sh.n_cand, n_app = sh.n_app;
    if (sh.error) return;
    if (n_cand == 0 || n_app == 0) break; // decoder.py:263-265, 285-287
    const u32 row_base = sh.flog_n;
    snapshot<BLOCK>(C, sh, (u32)rounds, C.flog_info + fbase, n_app, row_base);
    __syncthreads();
    if (threadIdx.x == 0) sh.flog_n = row_base + n_app;
    __syncthreads();
    if (sh.error) return;
    fbase = row_base;
    nf = n_app;
  }
  __syncthreads();
}

// Radix select over 64-bit keys (MSD, 8-bit digits, starting below the
// highest bit where the bounds [lo, hi] of all candidate keys differ).
// Returns t with count(key < t) < need <= count(key <= t).  On return
// `exact` tells whether ties at t still have to be resolved (then `need` is
// the number of keys equal to t that survive); otherwise every key <= t
// survives.
template <int BLOCK, typename KeyFn>
__device__ u64 radix_select(Shared &sh, u32 n, KeyFn keyf, u64 lo, u64 hi, u32 &need,
                            bool &exact) {
  const int tid = threadIdx.x;
  exact = true;
  if (lo == hi) return lo;
  int pos = 63 - __clzll(lo ^ hi);
  u64 prefix = pos >= 63 ? 0ull : (lo & ~((1ull << (pos + 1)) - 1));
  while (true) {
    const int lowbit = pos >= 7 ? pos - 7 : 0;
    const int nb = pos - lowbit + 1;
    const u64 above = pos >= 63 ? 0ull : ~((1ull << (pos + 1)) - 1);
    for (int b = tid; b < 256; b += BLOCK) sh.hist[b] = 0;
    __syncthreads();
    for (u32 i = tid; i < n; i += BLOCK) {
      bool ok;
      const u64 kk = keyf(i, ok);
      if (ok && (kk & above) == prefix) atomicAdd(&sh.hist[(kk >> lowbit) & ((1u << nb) - 1)], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      u32 cum = 0, b = 0;
      const u32 nbk = 1u << nb;
      for (; b < nbk; ++b) {
        if (cum + sh.hist[b] >= need) break;
        cum += sh.hist[b];
      }
      if (b >= nbk) b = nbk - 1; // unreachable when need <= matching keys
      sh.sel = b;
      sh.cum = cum;
    }
    __syncthreads();
    const u32 b = sh.sel;
    need -= sh.cum;
    const u32 cnt = sh.hist[b];
    __syncthreads();
    prefix |= ((u64)b << lowbit);
    if (lowbit == 0) {
      exact = cnt != need;
      return prefix;
    }
    if (cnt == need) {
      exact = false;
      return prefix | ((1ull << lowbit) - 1); // the whole bucket survives
    }
    pos = lowbit - 1;
  }
}

// _prune (decoder.py:319-334) + _best_token_pos (337-338) + silence bookkeeping
// (400-407).  Survivors are written to the token list.
template <int BLOCK, typename W, typename S>
__device__ void prune(const Chan<W, S> &C, Shared &sh) {
  const DecodeParams &P = *C.P;
  const int tid = threadIdx.x;
  const u32 n_all = min(sh.n_all, P.table_cap);
  u64 m = ~0ull;
  for (u32 i = tid; i < n_all; i += BLOCK) {
    u64 ck;
    u32 g, info;
    ld_cg_value(&C.table[C.all_list[i]], ck, g, info);
    m = min(m, ck);
  }
  const u64 best_ck = block_min_u64<BLOCK>(m, sh.redk);
  const double thr = key_cost(best_ck) + P.beam;
  const u64 thr_ck = cost_key(thr);
  if (tid == 0) sh.n_keep = 0;
  __syncthreads();
  u64 bk = ~0ull;
  u32 bs = 0xFFFFFFFFu;
  int bi = -1;
  for (u32 i = tid; i < n_all; i += BLOCK) {
    const u32 slot = C.all_list[i];
    Entry *e = &C.table[slot];
    u64 ck;
    u32 g, info;
    ld_cg_value(e, ck, g, info);
    if (ck <= thr_ck) {
      const u32 st = (u32)ld_cg_u64(&e->key);
      const u32 p = atomicAdd(&sh.n_keep, 1u);
      C.scr_key[p] = ck;
      C.scr_slot[p] = slot;
      if (ck < bk || (ck == bk && st < bs)) bk = ck, bs = st, bi = (int)slot;
    }
  }
  __syncthreads();
  const u32 n_keep = sh.n_keep;
  block_argmin<BLOCK>(bk, bs, bi, sh.redk, sh.reds, sh.redi);
  u64 tc = ~0ull;
  u32 ts = 0xFFFFFFFFu;
  if (n_keep > (u32)P.max_active) {
    u32 need = (u32)P.max_active;
    auto kf = [&](u32 i, bool &ok) -> u64 {
      ok = true;
      return C.scr_key[i];
    };
    bool exact;
    tc = radix_select<BLOCK>(sh, n_keep, kf, best_ck, thr_ck, need, exact);
    if (exact) {
      // ties at the threshold cost: the smallest states survive
      auto sf = [&](u32 i, bool &ok) -> u64 {
        ok = C.scr_key[i] == tc;
        return ok ? (u64)(u32)ld_cg_u64(&C.table[C.scr_slot[i]].key) : 0ull;
      };
      bool exact2;
      ts = (u32)radix_select<BLOCK>(sh, n_keep, sf, 0ull, 0xFFFFFFFFull, need, exact2);
    }
  }
  if (tid == 0) {
    sh.n_tok = 0;
    sh.max_depth = 0;
  }
  __syncthreads();
  int md = 0;
  for (u32 i = tid; i < n_keep; i += BLOCK) {
    const u64 ck = C.scr_key[i];
    const u32 slot = C.scr_slot[i];
    bool keep = ck < tc;
    u32 st = 0;
    if (!keep && ck == tc) {
      st = (u32)ld_cg_u64(&C.table[slot].key);
      keep = st <= ts;
    }
    if (keep) {
      Entry *e = &C.table[slot];
      if (!st) st = (u32)ld_cg_u64(&e->key);
      const u32 p = atomicAdd(&sh.n_tok, 1u);
      const TokInfo ti = C.flog_info[e->flog];
      md = max(md, ti.depth);
      C.tok_state[p] = st;
      C.tok_cost[p] = key_cost(ck);
      C.tok_info[p] = ti;
    }
  }
  atomicMax(&sh.max_depth, md);
  __syncthreads();
  if (tid == 0) {
    C.cs->max_depth = sh.max_depth;
    C.cs->info.num_active = (int)sh.n_tok;
    const TokInfo bti = C.flog_info[C.table[bi].flog];
    if (P.silence_ilabel > 0 && bti.last_il == P.silence_ilabel)
      C.cs->info.trailing_silence += 1;
    else
      C.cs->info.trailing_silence = 0;
  }
  __syncthreads();
}

// Writes the current token table = every slot claimed in this epoch
// (used after the utterance-start closure, which is not pruned).
template <int BLOCK, typename W, typename S>
__device__ void table_to_tokens(const Chan<W, S> &C, Shared &sh) {
  const u32 n_all = min(sh.n_all, C.P->table_cap);
  if (threadIdx.x == 0) sh.max_depth = 0;
  __syncthreads();
  int md = 0;
  for (u32 i = threadIdx.x; i < n_all; i += BLOCK) {
    Entry *e = &C.table[C.all_list[i]];
    u64 ck;
    u32 g, info;
    ld_cg_value(e, ck, g, info);
    const TokInfo ti = C.flog_info[e->flog];
    md = max(md, ti.depth);
    C.tok_state[i] = (u32)ld_cg_u64(&e->key);
    C.tok_cost[i] = key_cost(ck);
    C.tok_info[i] = ti;
  }
  atomicMax(&sh.max_depth, md);
  __syncthreads();
  if (threadIdx.x == 0) {
    C.cs->info.num_active = (int)n_all;
    C.cs->max_depth = sh.max_depth;
  }
  __syncthreads();
}

// Puts the utterance-start token into a fresh epoch (decoder.py:243-247).
template <int BLOCK, typename W, typename S>
__device__ void materialize_start(Chan<W, S> &C, Shared &sh) {
  const DecodeParams &P = *C.P;
  if (threadIdx.x == 0) {
    C.cs->epoch += 1;
    sh.n_all = 0;
    sh.n_app = 0;
    sh.flog_n = 1;
  }
  __syncthreads();
  C.epoch = C.cs->epoch;
  if (threadIdx.x == 0) {
    relax(C, sh, (u32)P.start, cost_key(0.0), 0xFFFFFFFFu, 0u, 0u);
    const u32 slot = C.all_list[0];
    TokInfo t;
    t.bp = -1;
    t.depth = 0;
    t.hits = 0;
    t.last_il = 0;
    C.flog_state[0] = (u32)P.start;
    C.flog_cost[0] = 0.0;
    C.flog_info[0] = t;
    C.table[slot].flog = 0;
  }
  __syncthreads();
}

// Copying collector for the emission arena: records reachable from the token
// list move to the other half in arena order (ids stay monotone), everything
// else (records of pruned or superseded tokens) is dropped.  Words never
// change: only record ids do, so the prefix-sharing path is reset.
template <int BLOCK, typename W, typename S>
__device__ void gc_arena(Chan<W, S> &C, Shared &sh) {
  const u32 n = sh.rec_n;
  const u32 nw = (n + 31) / 32;
  const u32 n_tok = (u32)C.cs->info.num_active;
  for (u32 w = threadIdx.x; w < nw; w += BLOCK) C.gc_bits[w] = 0;
  __syncthreads();
  for (u32 i = threadIdx.x; i < n_tok; i += BLOCK) {
    int r = C.tok_info[i].bp;
    while (r >= 0) {
      const u32 m = 1u << (r & 31);
      const u32 old = atomicOr(&C.gc_bits[r >> 5], m);
      if (old & m) break;
      r = C.arena[r].y;
    }
  }
  __syncthreads();
  u32 carry = 0;
  for (u32 base = 0; base < nw; base += BLOCK) {
    const u32 w = base + threadIdx.x;
    const u32 c = w < nw ? __popc(C.gc_bits[w]) : 0u;
    u32 total;
    const u32 ex = block_excl_scan<BLOCK>(c, total, sh.scan);
    if (w < nw) C.gc_rank[w] = carry + ex;
    carry += total;
  }
  __syncthreads();
  auto newid = [&](int i) -> int {
    const u32 w = (u32)i >> 5;
    return (int)(C.gc_rank[w] + __popc(C.gc_bits[w] & ((1u << (i & 31)) - 1u)));
  };
  for (u32 w = threadIdx.x; w < nw; w += BLOCK) {
    u32 b = C.gc_bits[w];
    while (b) {
      const int bit = __ffs(b) - 1;
      b &= b - 1;
      const int i = (int)(w * 32 + bit);
      const int2 r = C.arena[i];
      C.arena_to[newid(i)] = make_int2(r.x, r.y >= 0 ? newid(r.y) : -1);
    }
  }
  __syncthreads();
  for (u32 i = threadIdx.x; i < n_tok; i += BLOCK) {
    const int bp = C.tok_info[i].bp;
    if (bp >= 0) C.tok_info[i].bp = newid(bp);
  }
  __syncthreads();
  int2 *t = C.arena;
  C.arena = C.arena_to;
  C.arena_to = t;
  if (threadIdx.x == 0) {
    sh.rec_n = carry;
    C.cs->arena_half ^= 1;
    C.cs->path_len = 0;
  }
  __syncthreads();
}

// advance_frame (decoder.py:341-411) for frame row C.row.
template <int BLOCK, typename W, typename S>
__device__ void advance(Chan<W, S> &C, Shared &sh) {
  const DecodeParams &P = *C.P;
  ChanState *cs = C.cs;
  if (cs->info.status != AB_IDLE && cs->info.status != AB_DECODING) {
    if (threadIdx.x == 0) set_error(sh, E_STATUS);
    __syncthreads();
    return;
  }
  // one frame appends at most flog_cap records: collect first if they might not fit
  if (!cs->info.fresh && (unsigned long long)sh.rec_n + P.flog_cap > P.arena_cap) {
    gc_arena<BLOCK>(C, sh);
    if ((unsigned long long)sh.rec_n + P.flog_cap > P.arena_cap) {
      if (threadIdx.x == 0) set_error(sh, E_CAP);
      __syncthreads();
      return;
    }
  }
  if (cs->info.fresh) {
    materialize_start<BLOCK>(C, sh);
    epsilon_rounds<BLOCK>(C, sh, 0u, 1u); // utterance-start closure, no prune
    if (sh.error) return;
    table_to_tokens<BLOCK>(C, sh);
    if (threadIdx.x == 0) cs->info.fresh = 0;
  }
  __syncthreads();
  const u32 n_tok = (u32)cs->info.num_active;
  __syncthreads();
  if (threadIdx.x == 0) {
    cs->info.status = AB_DECODING;
    cs->epoch += 1;
    sh.n_all = 0;
    sh.n_app = 0;
    sh.n_cand = 0;
    sh.flog_n = 0;
  }
  __syncthreads();
  C.epoch = cs->epoch;
  expand<BLOCK, true>(C, sh, C.tok_state, C.tok_cost, n_tok, 0u);
  __syncthreads();
  if (sh.error) return;
  const u32 n_app = sh.n_app;
  if (n_app == 0) {
    // no emitting arcs: every token dies (decoder.py:394-398)
    if (threadIdx.x == 0) cs->info.num_active = 0;
  } else {
    snapshot<BLOCK>(C, sh, 0u, C.tok_info, n_app, 0u);
    __syncthreads();
    if (threadIdx.x == 0) sh.flog_n = n_app;
    __syncthreads();
    if (sh.error) return;
    epsilon_rounds<BLOCK>(C, sh, 0u, n_app);
    if (sh.error) return;
    prune<BLOCK>(C, sh);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    cs->info.frame_index += 1;
    cs->info.total_frames += 1;
  }
  __syncthreads();
}

// Traceback with prefix sharing against the channel's previous hypothesis
// path (EmissionStore.backtrace, decoder.py:95-102), then hypothesis output.
template <int BLOCK, typename W, typename S>
__device__ void emit_hyp(Chan<W, S> &C, Shared &sh, int out_idx, int kind, int fallback,
                         double cost, int bp, int depth, int hits) {
  const DecodeParams &P = *C.P;
  ChanState *cs = C.cs;
  if (threadIdx.x == 0) {
    int shared_words = 0;
    if ((u32)depth > P.path_cap) {
      set_error(sh, E_CAP);
    } else {
      int rec = bp, d = depth;
      const int plen = cs->path_len;
      while (d > 0) {
        if (d <= plen && C.path_rec[d - 1] == rec) break;
        C.path_rec[d - 1] = rec;
        const int2 r = C.arena[rec];
        C.path_words[d - 1] = r.x;
        rec = r.y;
        --d;
      }
      shared_words = d;
      cs->path_len = depth;
      const long long need = depth - shared_words;
      const long long off = P.words_used[blockIdx.x];
      if (off + need > P.words_stride || out_idx >= P.hyp_stride) set_error(sh, E_CAP);
      else P.words_used[blockIdx.x] = off + need;
      sh.shared_words = shared_words;
      sh.words_off = (long long)blockIdx.x * P.words_stride + off;
    }
  }
  __syncthreads();
  if (sh.error) return;
  const int s0 = sh.shared_words;
  const long long off = sh.words_off;
  for (int i = s0 + threadIdx.x; i < depth; i += BLOCK) P.words[off + (i - s0)] = C.path_words[i];
  if (threadIdx.x == 0) {
    DevHyp h;
    h.cost = cost;
    h.frame = cs->info.total_frames;
    h.kind = kind;
    h.fallback = fallback;
    h.hits = hits;
    h.shared = s0;
    h.n_words = depth;
    h.pad = 0;
    h.words_off = off;
    P.hyps[(size_t)blockIdx.x * P.hyp_stride + out_idx] = h;
  }
  __syncthreads();
}

// partial_hypothesis (decoder.py:414-423).
template <int BLOCK, typename W, typename S>
__device__ void partial(Chan<W, S> &C, Shared &sh, int out_idx) {
  ChanState *cs = C.cs;
  if (cs->info.fresh) {
    emit_hyp<BLOCK>(C, sh, out_idx, AB_PARTIAL, 0, 0.0, -1, 0, 0);
    return;
  }
  const u32 n = (u32)cs->info.num_active;
  if (n == 0) {
    if (threadIdx.x == 0) set_error(sh, E_DEAD);
    __syncthreads();
    return;
  }
  u64 bk = ~0ull;
  u32 bs = 0xFFFFFFFFu;
  int bi = -1;
  for (u32 i = threadIdx.x; i < n; i += BLOCK) {
    const u64 k = cost_key(C.tok_cost[i]);
    const u32 s = C.tok_state[i];
    if (k < bk || (k == bk && s < bs)) bk = k, bs = s, bi = (int)i;
  }
  block_argmin<BLOCK>(bk, bs, bi, sh.redk, sh.reds, sh.redi);
  const TokInfo t = C.tok_info[bi];
  emit_hyp<BLOCK>(C, sh, out_idx, AB_PARTIAL, 0, C.tok_cost[bi], t.bp, t.depth, t.hits);
}

// finalize (decoder.py:426-460): best final token by (cost + final, state),
// falling back to the best token; then the utterance is reset.
template <int BLOCK, typename W, typename S>
__device__ void finalize(Chan<W, S> &C, Shared &sh, int out_idx) {
  const DecodeParams &P = *C.P;
  ChanState *cs = C.cs;
  const int st = cs->info.status;
  if (st != AB_DECODING && st != AB_ENDPOINTED && !(st == AB_IDLE && cs->info.fresh)) {
    if (threadIdx.x == 0) set_error(sh, E_STATUS);
    __syncthreads();
    return;
  }
  __syncthreads();
  if (cs->info.fresh) {
    // zero-frame utterance: only the bare start token (no closure)
    if (threadIdx.x == 0) {
      TokInfo t;
      t.bp = -1;
      t.depth = 0;
      t.hits = 0;
      t.last_il = 0;
      C.tok_state[0] = (u32)P.start;
      C.tok_cost[0] = 0.0;
      C.tok_info[0] = t;
      cs->info.num_active = 1;
      cs->info.fresh = 0;
    }
    __syncthreads();
  }
  const u32 n = (u32)cs->info.num_active;
  if (n == 0) {
    if (threadIdx.x == 0) set_error(sh, E_DEAD);
    __syncthreads();
    return;
  }
  u64 fk = ~0ull, bk = ~0ull;
  u32 fs = 0xFFFFFFFFu, bs = 0xFFFFFFFFu;
  int fi = -1, bi = -1;
  for (u32 i = threadIdx.x; i < n; i += BLOCK) {
    const double c = C.tok_cost[i];
    const u32 s = C.tok_state[i];
    const u64 k = cost_key(c);
    if (k < bk || (k == bk && s < bs)) bk = k, bs = s, bi = (int)i;
    const double fc = __ldg(&P.final_cost[s]);
    if (fc == fc) { // final state
      const u64 tk = cost_key(c + fc);
      if (tk < fk || (tk == fk && s < fs)) fk = tk, fs = s, fi = (int)i;
    }
  }
  block_argmin<BLOCK>(fk, fs, fi, sh.redk, sh.reds, sh.redi);
  block_argmin<BLOCK>(bk, bs, bi, sh.redk, sh.reds, sh.redi);
  int b;
  int fallback;
  double cost;
  if (fi >= 0) {
    b = fi;
    fallback = 0;
    cost = C.tok_cost[b] + __ldg(&P.final_cost[C.tok_state[b]]);
  } else {
    b = bi;
    fallback = 1;
    cost = C.tok_cost[b];
  }
  const TokInfo t = C.tok_info[b];
  emit_hyp<BLOCK>(C, sh, out_idx, AB_FINAL, fallback, cost, t.bp, t.depth, t.hits);
  if (sh.error) return;
  if (threadIdx.x == 0) {
    // _reset_utterance (decoder.py:151-159)
    cs->info.num_active = 0;
    cs->info.fresh = 1;
    cs->info.frame_index = 0;
    cs->info.trailing_silence = 0;
    sh.rec_n = 0;
    sh.rec_logical = 0;
    cs->path_len = 0;
    cs->max_depth = 0;
    cs->info.utterance_index += 1;
    cs->info.status = AB_IDLE;
  }
  __syncthreads();
}

template <int BLOCK, typename W, typename S>
__device__ void setup_channel(Chan<W, S> &C, const DecodeParams &P, int slot, S *sh_row,
                              u32 *sh_ctx) {
  C.P = &P;
  C.slot = slot;
  C.cs = &P.chans[slot];
  const size_t s = (size_t)slot;
  C.table = P.table + s * P.table_cap;
  C.tok_state = P.tok_state + s * P.tok_cap;
  C.tok_cost = P.tok_cost + s * P.tok_cap;
  C.tok_info = P.tok_info + s * P.tok_cap;
  C.flog_state = P.flog_state + s * P.flog_cap;
  C.flog_cost = P.flog_cost + s * P.flog_cap;
  C.flog_info = P.flog_info + s * P.flog_cap;
  C.all_list = P.all_list + s * P.table_cap;
  C.app_list = P.app_list + s * P.table_cap;
  C.scr_key = P.scr_key + s * P.table_cap;
  C.scr_slot = P.scr_slot + s * P.table_cap;
  C.arena = P.arena + (2 * s + (C.cs->arena_half & 1)) * P.arena_cap;
  C.arena_to = P.arena + (2 * s + ((C.cs->arena_half & 1) ^ 1)) * P.arena_cap;
  C.gc_bits = P.gc_bits + s * (P.arena_cap / 32 + 1);
  C.gc_rank = P.gc_rank + s * (P.arena_cap / 32 + 1);
  C.path_rec = P.path_rec + s * P.path_cap;
  C.path_words = P.path_words + s * P.path_cap;
  C.row = sh_row;
  C.epoch = C.cs->epoch;
  const int h = C.cs->info.context;
  C.ctx_mode = 0;
  C.discount = 0.0;
  if (h >= 0 && h < P.num_ctxs) {
    const CtxDesc d = P.ctxs[h];
    C.discount = d.discount;
    C.ctx_k = d.k;
    if (d.k == 0) {
      C.ctx_mode = 0;
    } else if (d.mode == AB_CTX_BITSET) {
      C.ctx_mode = 3;
      C.ctx_bits = d.bits;
    } else if (d.k <= (u32)CTX_SMEM_MAX) {
      for (u32 i = threadIdx.x; i < d.k; i += BLOCK) sh_ctx[i] = d.list[i];
      C.ctx_mode = 1;
      C.ctx_list = sh_ctx;
    } else {
      C.ctx_mode = 2;
      C.ctx_list = d.list;
    }
  }
  __syncthreads();
}

template <int BLOCK, typename W, typename S>
__global__ void __launch_bounds__(BLOCK) decode_kernel(const DecodeParams P) {
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  __shared__ Shared sh;
  u32 *sh_ctx = reinterpret_cast<u32 *>(dyn_smem);
  S *sh_row = reinterpret_cast<S *>(dyn_smem + CTX_SMEM_MAX * sizeof(u32));
  const bool row_in_smem = (size_t)P.L * sizeof(S) <= (size_t)SCORE_SMEM_MAX_BYTES;
  const int slot = P.slots[blockIdx.x];
  Chan<W, S> C;
  setup_channel<BLOCK>(C, P, slot, sh_row, sh_ctx);
  ChanState *cs = C.cs;
  if (threadIdx.x == 0) {
    sh.error = 0;
    sh.rec_n = cs->rec_phys;
    sh.rec_logical = (unsigned long long)cs->info.store_len;
    sh.cnt_tok = sh.cnt_emit = sh.cnt_eps = 0;
    sh.n_all = sh.n_app = sh.n_cand = sh.flog_n = 0;
  }
  __syncthreads();
  const int T = P.frames[blockIdx.x];
  const S *scores = reinterpret_cast<const S *>(P.scores) + P.score_off[blockIdx.x];
  int n_out = 0;
  if (P.mode == AB_MODE_STREAM && cs->info.status == AB_FINISHED) {
    __syncthreads();
    if (threadIdx.x == 0) cs->info.status = AB_IDLE; // decoder.py:488-489
  }
  __syncthreads();
  int t = 0;
  for (; t < T; ++t) {
    if (P.mode == AB_MODE_STREAM) {
      // a frame adds at most 1 + max_eps words to any path and emits at most two
      // hypotheses; pause (the host relaunches) if they might not fit
      const long long bound = (long long)(cs->info.fresh ? 0 : cs->max_depth) + 2 + P.max_eps;
      if (P.words_used[blockIdx.x] + 2 * bound > P.words_stride || n_out + 2 > P.hyp_stride) break;
    }
    const S *grow = scores + (size_t)t * P.L;
    if (row_in_smem) {
      for (int i = threadIdx.x; i < P.L; i += BLOCK) sh_row[i] = grow[i];
      C.row = sh_row;
    } else {
      C.row = grow;
    }
    __syncthreads();
    advance<BLOCK>(C, sh);
    if (sh.error) break;
    if (P.mode == AB_MODE_STREAM) {
      if (cs->info.frame_index % P.partial_every == 0) {
        partial<BLOCK>(C, sh, n_out++);
        if (sh.error) break;
      }
      if (cs->info.trailing_silence >= P.endpoint_silence_frames) { // detect_endpoint 463-464
        __syncthreads();
        if (threadIdx.x == 0) cs->info.status = AB_ENDPOINTED;
        __syncthreads();
        finalize<BLOCK>(C, sh, n_out++);
        if (sh.error) break;
      }
    }
    __syncthreads();
  }
  const bool done = t == T;
  if (P.mode == AB_MODE_STREAM && !sh.error && done) {
    if (cs->info.frame_index > 0 || T == 0) finalize<BLOCK>(C, sh, n_out++);
    __syncthreads();
    if (!sh.error && threadIdx.x == 0) cs->info.status = AB_FINISHED;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    cs->rec_phys = sh.rec_n;
    cs->info.store_len = (long long)sh.rec_logical;
    cs->info.tok_expansions += sh.cnt_tok;
    cs->info.emit_arcs += sh.cnt_emit;
    cs->info.eps_arcs += sh.cnt_eps;
    cs->info.error = sh.error;
    P.n_hyps[blockIdx.x] = n_out;
    P.errors[blockIdx.x] = sh.error;
    P.frames_done[blockIdx.x] = t;
  }
}

// Standalone partial / finalize for one channel (the per-call Python API).
template <int BLOCK, typename W, typename S>
__global__ void __launch_bounds__(BLOCK) hyp_kernel(const DecodeParams P, int which) {
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  __shared__ Shared sh;
  u32 *sh_ctx = reinterpret_cast<u32 *>(dyn_smem);
  S *sh_row = reinterpret_cast<S *>(dyn_smem + CTX_SMEM_MAX * sizeof(u32));
  Chan<W, S> C;
  setup_channel<BLOCK>(C, P, P.slots[blockIdx.x], sh_row, sh_ctx);
  if (threadIdx.x == 0) {
    sh.error = 0;
    sh.rec_n = C.cs->rec_phys;
    sh.rec_logical = (unsigned long long)C.cs->info.store_len;
  }
  __syncthreads();
  if (which == AB_PARTIAL) partial<BLOCK>(C, sh, 0);
  else finalize<BLOCK>(C, sh, 0);
  __syncthreads();
  if (threadIdx.x == 0) {
    C.cs->rec_phys = sh.rec_n;
    C.cs->info.store_len = (long long)sh.rec_logical;
    P.n_hyps[blockIdx.x] = sh.error ? 0 : 1;
    P.errors[blockIdx.x] = sh.error;
  }
}

} // namespace ab
