// Batched, frame-synchronous, biased token passing on sm_100a.
//
// One CTA owns one channel (a stream) for the whole call and runs every frame
// of it: score-row staging, emitting expansion with the fused boost lookup,
// bounded epsilon closure, beam + max_active pruning, partial / final
// traceback.  Channels are independent, so a launch of n
// CTAs decodes n channels with no inter-CTA synchronisation; with ~1000
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
//
// Per-frame data flow (all per channel):
//   token list --expand(emitting CSR)--> token table (128-bit CAS minimum);
//       every installed candidate owns a frontier row written before its CAS
//   rows of round r --expand(epsilon CSR)--> table ... (Jacobi rounds)
//   live frontier rows --prune (beam, exact top-k radix select)--> token list
//   survivors --resolve (source links)--> provenance + emission records
#pragma once
#include <cooperative_groups.h>
#include <cooperative_groups/scan.h>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/arcboost_b200.h"

namespace ab {

typedef unsigned long long u64;
typedef uint32_t u32;

constexpr u64 KEY_EPOCH_MASK = 0x7FFFFFFF00000000ull;
// value.info = epoch tag(13) | frontier row of the winner(19).  Rows are
// allocated in round order inside a frame, so the row also tells the round:
// a value whose row is below the current round's first row is from an earlier
// round (no round field, so the tag is wide: the table is wiped once per 8191
// epochs).
constexpr int TAG_SHIFT = 19;
constexpr u32 TAG_MASK = 0x1FFFu;
constexpr u32 VROW_MASK = (1u << TAG_SHIFT) - 1;
constexpr u32 MAX_ROWS = 1u << TAG_SHIFT;  // frontier rows per channel-frame
// arc records carry the destination's "has epsilon arcs" flag in bit 31 of the
// arc id; every candidate into one destination has the same flag, so the
// (cost, arc id) order inside a slot is unchanged (graphs have < 2^31 arcs)
constexpr u32 G_DEST_EPS = 0x80000000u;
constexpr u32 G_MASK = 0x7FFFFFFFu;
constexpr u32 G_START = 0xFFFFFFFFu; // frontier row of the utterance-start token
constexpr u32 MAX_TOKENS = 1u << 17;            // distinct tokens per channel-frame
constexpr u32 MAX_HASH_SLOTS = 1u << 22;        // hashed token-table slots per channel
// a row's state as read back: state | ecode (below) | DISP | DEAD
constexpr u32 ROW_DEAD = 0x80000000u;  // superseded by a later round (an application, not a token)
constexpr u32 ROW_DISP = 0x40000000u;  // displaced in its own round (not an application)
constexpr u32 ROW_STATE = 0x07FFFFFFu;
// DEAD / DISP live in a separate kill word per row, written once, by the
// thread whose CAS replaced the row, with the epoch tag: (tag << 2) | KW_*.
// No kill queue and no pass applying it, so a pass needs one barrier (the
// next pass's listing reads DISP behind it; DEAD is read by prune only).  The
// stored row state word carries ROW_REC at bit 30 (the row has an output
// label: an emission record unless displaced).
constexpr u32 KW_DEAD = 1u, KW_DISP = 2u;
constexpr u32 ROW_REC = 0x40000000u;
// a candidate's flags (registers; boost / output label also go to the row's aux word)
constexpr u32 ROW_EPS = 0x20000000u;   // the state has epsilon out-arcs
constexpr u32 ROW_BOOST = 0x10000000u; // the winning arc is boosted
constexpr u32 ROW_HASOL = 0x08000000u; // the winning arc has an output label (an emission record)
// Out-degree codes travel with a state (no per-expansion degree load): an arc
// record's next-state word is dest | ecode << 27 | xcode << 30 (ecode =
// emitting arcs 0..4, 7 = overflow; xcode = epsilon arcs 0..2, 3 = overflow);
// a frontier row's and a token's state word keep the ecode (bits 27-29, the
// row's DISP / DEAD flags are bits 30 / 31), an epsilon-frontier entry's the
// xcode (bits 27-28).
constexpr u32 CODE_SHIFT = 27;
constexpr u32 ECODE_MASK = 7u << CODE_SHIFT;
constexpr u32 ECODE_OVF = 7, XCODE_OVF = 3;
__device__ __forceinline__ u32 ecode_of(u32 dc) { return dc & 7u; }  // dc = record word >> 27
__device__ __forceinline__ u32 xcode_of(u32 dc) { return dc >> 3; }
// frontier row aux word {source | AUX_BOOST | AUX_HASOL, arc id}: the
// provenance walk reads one 8-byte word per step
constexpr u32 AUX_BOOST = 0x80000000u;
constexpr u32 AUX_HASOL = 0x40000000u;
constexpr u32 AUX_START = 0x20000000u; // the utterance-start row (no source arc)
constexpr u32 AUX_SRC = 0x1FFFFFFFu;
__device__ __forceinline__ u32 aux_src(u32 src, u32 rflags, u32 g) {
  return src | ((rflags & ROW_BOOST) ? AUX_BOOST : 0u) | ((rflags & ROW_HASOL) ? AUX_HASOL : 0u) |
         (g == G_START ? AUX_START : 0u);
}
constexpr int CTX_SMEM_WORDS = 4096;        // sparse contexts / label bitmaps (16 KB, sized per launch)
// Bloom filter (two hashes, 128 Kbit = 16 KB) of the states from which an
// epsilon path lowers a cost: the only states the cutoff's slack applies to
// (advance()).  False positives only keep a few more candidates.
#ifndef AB_NEG_WORDS
#define AB_NEG_WORDS 4096
#endif
constexpr u32 NEG_WORDS = AB_NEG_WORDS;
#ifndef AB_HQ_MIN_STATES
#define AB_HQ_MIN_STATES (24 * 1024)
#endif
constexpr size_t HQ_MIN_STATES = AB_HQ_MIN_STATES; // more such states: per-state slack instead
#ifndef AB_HQ_BITS
#define AB_HQ_BITS 8 // bits of per-state slack (2 or 8; 8 with the per-position flags: profiles/r02_hq_bits_ab.log)
#endif
constexpr u32 HQ_BITS = AB_HQ_BITS, HQ_PER_WORD = 32 / HQ_BITS, HQ_MAX = (1u << HQ_BITS) - 1;
__host__ __device__ __forceinline__ u32 hq_get(const u32 *hq, u32 s) {
  return (hq[s / HQ_PER_WORD] >> ((s % HQ_PER_WORD) * HQ_BITS)) & HQ_MAX;
}
constexpr int NEG_SHIFT = 32 - 5 - __builtin_ctz(NEG_WORDS); // hashes of log2(32 * NEG_WORDS) bits
// A context stores the filter at NEG_WORDS and folded to every smaller power
// of two down to NEG_MIN_WORDS (bit j of the half-size filter = OR of bits 2j,
// 2j+1: the hashes are top bits, one shift more per halving); a launch copies
// the smallest one that keeps ~8 bits per flagged state (the rest of shared
// memory stays L1).  The size-W filter is at word 2 NEG_WORDS - 2 W.
constexpr u32 NEG_MIN_WORDS = 256;
constexpr u32 NEG_BLOCK_WORDS = 2 * NEG_WORDS - NEG_MIN_WORDS;
__host__ __device__ __forceinline__ u32 neg_h1(u32 s) { return (s * 2654435761u) >> NEG_SHIFT; }
__host__ __device__ __forceinline__ u32 neg_h2(u32 s) { return ((s ^ (s >> 16)) * 0x85EBCA6Bu) >> NEG_SHIFT; }
__device__ __forceinline__ bool neg_test(const u32 *b, u32 s, u32 fold) {
  const u32 a = neg_h1(s) >> fold, c = neg_h2(s) >> fold;
  return ((b[a >> 5] >> (a & 31)) & (b[c >> 5] >> (c & 31)) & 1u) != 0;
}
constexpr int SCORE_SMEM_MAX_BYTES = 32768; // larger score rows are read from L2
constexpr u32 SLOT_E = 4, SLOT_X = 2;         // arc records per state slot (emitting / epsilon)
constexpr u32 DEG_OVF = 15;                   // degree nibble: arcs live in the overflow area
#ifndef AB_EXP_Q
#define AB_EXP_Q 2
#endif
#ifndef AB_WARP_TILES_MIN_BLOCK
#define AB_WARP_TILES_MIN_BLOCK 1024
#endif
// Frontier rows and epsilon entries are read back only after the rest of the
// pass: with many channels per SM (256-thread CTAs, DRAM-bound) they are
// stored evict-first so L2 keeps the token-table lines between load and CAS;
// a 1024-thread CTA (few channels, L2-resident working set) stores normally.
// A displaced row leaves the next round's epsilon frontier through its own
// DISP flag, read when the round lists its entries (the entry is not marked
// at kill time, so rows carry no epsilon-list position).
template <int BLOCK, typename T> __device__ __forceinline__ void st_row(T *p, T v) {
  if (BLOCK <= 256) __stcs(p, v);
  else *p = v;
}
// A frontier row's aux word {source | AUX flags, olabel, ilabel}: 8 bytes
// (labels packed 16:16) with 16-bit labels, else 16 (F::aux8); the pool is
// sized for 16 per row either way.
template <int BLOCK, typename F> __device__ __forceinline__ void store_aux(uint4 *aux, u32 row, u32 x, u32 ol, u32 il) {
  if constexpr (F::aux8) st_row<BLOCK>(reinterpret_cast<uint2 *>(aux) + row, make_uint2(x, (ol << 16) | il));
  else st_row<BLOCK>(aux + row, make_uint4(x, 0u, ol, il));
}
template <typename F> __device__ __forceinline__ void load_aux(const uint4 *aux, u32 row, u32 &x, u32 &ol, u32 &il);
template <typename F> __device__ __forceinline__ void load_aux(const uint4 *aux, u32 row, u32 &x, u32 &ol, u32 &il) {
  if constexpr (F::aux8) {
    const uint2 a = reinterpret_cast<const uint2 *>(aux)[row];
    x = a.x;
    ol = a.y >> 16;
    il = a.y & 0xFFFFu;
  } else {
    const uint4 a = aux[row];
    x = a.x;
    ol = a.z;
    il = a.w;
  }
}
#ifndef AB_EXP_Q1024
#define AB_EXP_Q1024 1 // 1024-thread CTAs: 32-input warp sub-tiles
#endif
#ifndef AB_EXP_Q256
#define AB_EXP_Q256 3 // 256-thread CTAs (many channels): larger tiles, fewer tile barriers
#endif
#ifndef AB_EXP_U
#define AB_EXP_U 1
#endif
// inputs per thread per expansion tile (the tile arrays are static shared
// memory: 20 bytes per input, under the 48 KB static limit at 1024 threads)
template <int BLOCK> __host__ __device__ constexpr int exp_q() {
  return BLOCK <= 256 ? AB_EXP_Q256 : (BLOCK >= 1024 ? AB_EXP_Q1024 : AB_EXP_Q);
}
constexpr int EXP_U = AB_EXP_U; // arcs per thread in flight (arc loads, table round trips)
// A cluster's channel (one 1024-thread CTA per SM, latency-bound): more arcs
// per thread in flight
#ifndef AB_EXP_U_CLUSTER
#define AB_EXP_U_CLUSTER 1 // (2 spills at 64 registers: slower, profiles/r02_c1_c2_phase_profile.log)
#endif
constexpr u32 TILE_COARSE = 128; // coarse search index entries (tiles of up to 4096 arcs)
#ifndef AB_PRUNE_Q
#define AB_PRUNE_Q 4
#endif
constexpr int PRUNE_Q = AB_PRUNE_Q; // rows per thread in flight (prune)
constexpr u32 RANK_MAX = 256; // prune's split bucket: selection by rank up to this many rows (else radix)

enum { CTX_NONE = 0, CTX_SLIST = 1, CTX_GLIST = 2, CTX_BITSET = 3, CTX_LABELS = 4 };
// LIST contexts of up to LIST_SMEM_MAX arcs: a two-hash Bloom filter of their
// ids in shared memory (32 bits per arc, rounded up to a power of two: false
// positives ~0.2%, so a warp rarely has a lane that goes further), and the
// ids as a hash set in global memory (load <= 1/2: one or two loads) probed
// for the filter's hits; larger lists probe the set alone.  Shared
// memory not taken stays L1 (the kernel is sensitive to it).
constexpr u32 LIST_SMEM_MAX = 2048;
__host__ __device__ __forceinline__ u32 list_b1(u32 g, u32 nbits) { return ((g * 2654435761u) >> 7) & (nbits - 1u); }
__host__ __device__ __forceinline__ u32 list_b2(u32 g, u32 nbits) { return ((g * 0x85EBCA6Bu) >> 9) & (nbits - 1u); }
__host__ __device__ __forceinline__ u32 list_slot(u32 g, u32 mask) { return ((g ^ (g >> 15)) * 0x2C1B3C6Du >> 8) & mask; }

// Token provenance carried with every token (decoder.py:58-62 + last_il 138).
struct __align__(16) TokInfo {
  int bp;      // emission-arena record id, -1 = utterance start
  int depth;   // words on the path (records reachable from bp)
  int hits;    // boosted arcs on the path
  int last_il; // ilabel of the last emitting arc (decoder.py:393, 404)
};

// Token table.  Hashed (graphs too large for a direct table in the memory
// budget): 32-B slots (one sector), key = state | epoch << 32, the frontier
// row of the slot's latest application, and the value.  Direct: one 16-B
// value per graph state (slot = state, no key, no probing) plus a u32 row
// array.  The value (16 B, the CAS-128 target) = ordered cost key, global arc
// id, info.  A value whose epoch tag differs from the channel's current tag is
// empty; the table is wiped when the 13-bit tag wraps (every 8191 epochs).
struct __align__(32) Entry {
  u64 key;
  u32 flog; // frontier-log row of the latest application in this frame
  u32 pad;
  u64 ck;
  u32 g;
  u32 info;
};

struct CtxDesc {
  double discount;
  u32 k;     // arcs in the context
  int mode;  // CTX_*
  u32 words; // CTX_LABELS: bitmap words
  u32 lmask; // list: hash set size - 1
  const u32 *list; // the arc ids as an open-addressing hash set (list_slot, ~0 = empty)
  const u32 *hash; // CTX_SLIST: Bloom filter of the ids (words words)
  const u32 *bits;   // CTX_BITSET: bit per emitting record position, CTX_LABELS: olabel bitmap
  const u32 *bits_x; // CTX_BITSET: bit per epsilon record position
  double slack;      // -min over states of the cheapest epsilon path from them (>= 0)
  int slack_rounds;  // slack bounds paths of at most this many epsilon arcs (INT_MAX: any)
  int pad2;
  const u32 *neg;    // NEG_BLOCK_WORDS: Bloom filters of the states where that path is negative
  // contexts with too many such states for the filter: per-state slack
  // ceil(-h(s) / hq_unit) in 2 bits (0 = none, 16 states per word: 1.25 MB
  // for 5M states, L2-resident), read for band candidates only
  const u32 *hq;
  double hq_unit;
  const u32 *fbits, *fbits_x; // with hq: per record position, "the destination's hq > 0"
};

// Arc record formats.  Fmt16: f32 weight, 16-bit labels (one 16 B load).
// Fmt24: f64 weight and 32-bit labels.  Records of a state are contiguous
// and in source order (their g increase).
struct __align__(16) EArc16 { u32 ns, g; float w; u32 lab; };
struct __align__(16) XArc16 { u32 ns, g; float w; u32 ol; };
struct __align__(8) EArc24 { u32 ns, g, il, ol; double w; };
struct __align__(8) XArc24 { u32 ns, g, ol, pad; double w; };

template <bool H, bool SMT = false> struct Fmt16 {
  static constexpr bool hashed = H; // token table: hashed (true) or identity-mapped
  static constexpr bool smem_table = SMT; // identity-mapped table in shared memory (small graphs)
  static constexpr int cluster = 1;       // CTAs per channel
  static constexpr bool aux8 = true;      // 8-byte frontier-row aux (16-bit labels)
  typedef EArc16 E;
  typedef XArc16 X;
  static __device__ __forceinline__ void emit(const void *base, u32 a, u32 &ns, u32 &g, double &w,
                                              u32 &il, u32 &ol) {
    const uint4 r = __ldg(reinterpret_cast<const uint4 *>(base) + a);
    ns = r.x;
    g = r.y;
    w = (double)__uint_as_float(r.z);
    il = r.w & 0xFFFFu;
    ol = r.w >> 16;
  }
  static __device__ __forceinline__ void eps(const void *base, u32 a, u32 &ns, u32 &g, double &w,
                                             u32 &ol) {
    const uint4 r = __ldg(reinterpret_cast<const uint4 *>(base) + a);
    ns = r.x;
    g = r.y;
    w = (double)__uint_as_float(r.z);
    ol = r.w;
  }
};
template <bool H> struct Fmt24 {
  static constexpr bool hashed = H;
  static constexpr bool smem_table = false;
  static constexpr int cluster = 1;
  static constexpr bool aux8 = false;
  typedef EArc24 E;
  typedef XArc24 X;
  static __device__ __forceinline__ void emit(const void *base, u32 a, u32 &ns, u32 &g, double &w,
                                              u32 &il, u32 &ol) {
    // 24-byte records are only 8-byte aligned: three 8-byte loads
    const EArc24 *p = reinterpret_cast<const EArc24 *>(base) + a;
    const uint2 r0 = __ldg(reinterpret_cast<const uint2 *>(p));
    const uint2 r1 = __ldg(reinterpret_cast<const uint2 *>(p) + 1);
    ns = r0.x;
    g = r0.y;
    il = r1.x;
    ol = r1.y;
    w = __ldg(&p->w);
  }
  static __device__ __forceinline__ void eps(const void *base, u32 a, u32 &ns, u32 &g, double &w,
                                             u32 &ol) {
    const XArc24 *p = reinterpret_cast<const XArc24 *>(base) + a;
    const uint2 r0 = __ldg(reinterpret_cast<const uint2 *>(p));
    ns = r0.x;
    g = r0.y;
    ol = __ldg(&p->ol);
    w = __ldg(&p->w);
  }
};

typedef Fmt16<false, true> Fmt16S; // direct table in shared memory (one macro argument)
// A channel decoded by a cluster of CL CTAs (C1 / C2: few channels, small
// graph): the shared-memory table split across the cluster (state s in CTA
// s % CL), the channel's counters in the leader's shared memory, DSMEM between.
template <int CL> struct Fmt16SC : Fmt16<false, true> {
  static constexpr int cluster = CL;
};
typedef Fmt16SC<2> Fmt16SC2;
typedef Fmt16SC<4> Fmt16SC4;
typedef Fmt16SC<8> Fmt16SC8;
typedef Fmt16SC<16> Fmt16SC16; // (non-portable cluster size)
template <typename F> __host__ __device__ constexpr int exp_u() { return F::cluster > 1 ? AB_EXP_U_CLUSTER : EXP_U; }

struct ChanState {
  ab_channel_info info; // info.store_len = records appended this utterance (reference len(store))
  u32 epoch;
  int path_len;
  int max_depth;  // deepest token path in the current token list
  int arena_half; // which half of the channel's arena is live (copying GC)
  u32 rec_phys;   // records physically in the live half
  u32 tok_half;   // which half of the channel's token-provenance buffer is current
  double prev_best; // best token cost of the previous frame (cost histogram window)
  double prev_cut;  // the previous frame's pruning cutoff (inf: none yet), see advance()
  double cut_rise;  // recent rise of the cutoff per frame (decaying maximum)
  int best_tok;     // token-list index of the best (cost, state) token from prune, -1 = unknown
};

struct DevHyp {
  double cost;
  long long frame;
  int kind, fallback, hits, shared, n_words, pad;
  long long words_off;
};

struct DecodeParams {
  // graph (device CSR split into emitting / epsilon arcs, fst.py:116-191)
  const uint2 *e_rng; // per state {begin, end} of its emitting arcs
  const void *e_arcs;
  const uint2 *x_rng; // per state {begin, end} of its epsilon arcs
  const void *x_arcs;
  // per state: emitting arc count (low nibble), epsilon arc count (high
  // nibble); DEG_OVF = more than a slot holds, use the ranges.  A state with
  // at most SLOT_E emitting (SLOT_X epsilon) arcs has them at s * SLOT_E
  // (s * SLOT_X): no range lookup.  1 byte per state stays L2-resident.
  const unsigned char *deg;
  const double *final_cost; // NaN = not final
  int start;
  int num_states;
  unsigned long long *prof; // phase cycle counters (AB_PROFILE builds only)
  int L;
  const CtxDesc *ctxs;
  int num_ctxs;
  // per-channel pools (slot-major)
  ChanState *chans;
  Entry *table;   // hashed
  u64 *vals;      // direct: [channel][table_cap][2]
  u32 table_cap, table_mask, hash_shift;
  int hashed;
  u32 *tok_state;
  double *tok_cost;
  TokInfo *tok_info;
  u32 tok_cap;
  u32 *flog_state;
  u64 *flog_ck;
  uint4 *flog_aux; // {source | AUX flags, olabel, ilabel} per frontier row (store_aux)
  uint4 *eps_list; // [channel][flog_cap] {row, state | flags, cost key}: rows whose state has
                   // epsilon arcs, in write order (the next round's frontier)
  u32 flog_cap;
  u32 *app_list;  // [channel][flog_cap] prune scratch (split-bucket row states)
  u32 *flog_kill; // [channel][flog_cap] kill words (KW_*)
  u64 *scr_key;
  u32 *scr_row;
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
  const int *frames;        // frames of this launch
  const int *stream_frames; // frames of the whole ab_decode call (chunked host staging)
  const long long *score_off;
  const void *scores;
  int mode;
  int final_chunk; // stream mode: the frames of this launch end the streams (finalize)
  // expansion-time cutoff (advance()): off when exact; slack of unbiased
  // decoding; hint = previous cutoff + max(rise, hint_min) + hint_extra
  int exact;
  double slack0, hint_min, hint_extra;
  // an utterance's first frames (token set still growing, the cutoff's rise
  // irregular) get hint_warm more margin
  double hint_warm;
  int hint_warm_frames;
  int slack0_rounds;
  const u32 *neg0; // NEG_WORDS bitmap of the unbiased graph
  // dynamic shared memory layout (host: launch_smem_layout)
  u32 ctx_words_cap; // context words in shared memory (LABELS bitmap / LIST arcs)
  u32 neg_words;     // 0 or the neg Bloom filter's words (a power of two <= NEG_WORDS) after the score row
  int row_in_smem;   // the frame's score row is staged in shared memory (else read through L1)
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

// whole 32-byte hashed entry in one request (key and value)
__device__ __forceinline__ void ld_cg_entry(const Entry *e, u64 &key, u64 &ck, u32 &g, u32 &info) {
  u64 a, b, c, d;
  asm volatile("ld.global.cg.v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(e));
  asm volatile("" ::"l"(b)); // the entry's row field is not needed here
  key = a;
  ck = c;
  g = (u32)d;
  info = (u32)(d >> 32);
}
// Value accessors; SM = where the table lives: 0 global memory, 1 this CTA's
// shared memory (Fmt::smem_table), 2 the cluster's distributed shared memory
// (generic addresses into the peer CTAs' windows, Fmt::cluster > 1).
template <typename F> __host__ __device__ constexpr int table_space() {
  return F::smem_table ? (F::cluster > 1 ? 2 : 1) : 0;
}
template <int SM = 0> __device__ __forceinline__ void ld_cg_value(const u64 *v, u64 &ck, u32 &g, u32 &info) {
  u64 a, b;
  if (SM == 1) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(v);
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(sa) : "memory");
  } else if (SM == 2) {
    asm volatile("ld.relaxed.cluster.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(v) : "memory");
  } else {
    asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(v));
  }
  ck = a;
  g = (u32)b;
  info = (u32)(b >> 32);
}
// CAS-128 that only issues: the old value comes back in (r0, r1); the caller
// compares, so several can be in flight per thread.
template <int SM = 0>
__device__ __forceinline__ void cas128(u64 *addr, u64 e0, u64 e1, u64 d0, u64 d1, u64 &r0, u64 &r1) {
  if (SM == 2) {
    asm volatile(
        "{\n .reg .b128 e, d, r;\n mov.b128 e, {%2, %3};\n mov.b128 d, {%4, %5};\n"
        " atom.relaxed.cluster.cas.b128 r, [%6], e, d;\n mov.b128 {%0, %1}, r;\n}\n"
        : "=l"(r0), "=l"(r1)
        : "l"(e0), "l"(e1), "l"(d0), "l"(d1), "l"(addr)
        : "memory");
  } else if (SM == 1) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(addr);
    asm volatile(
        "{\n .reg .b128 e, d, r;\n mov.b128 e, {%2, %3};\n mov.b128 d, {%4, %5};\n"
        " atom.shared.cas.b128 r, [%6], e, d;\n mov.b128 {%0, %1}, r;\n}\n"
        : "=l"(r0), "=l"(r1)
        : "l"(e0), "l"(e1), "l"(d0), "l"(d1), "r"(sa)
        : "memory");
  } else {
    asm volatile(
        "{\n .reg .b128 e, d, r;\n mov.b128 e, {%2, %3};\n mov.b128 d, {%4, %5};\n"
        " atom.global.cas.b128 r, [%6], e, d;\n mov.b128 {%0, %1}, r;\n}\n"
        : "=l"(r0), "=l"(r1)
        : "l"(e0), "l"(e1), "l"(d0), "l"(d1), "l"(addr)
        : "memory");
  }
}

// 128-bit compare-and-swap on the value half of an entry (ATOMG.E.CAS.128).
template <int SM = 0>
__device__ __forceinline__ bool cas_value(u64 *v, u64 &ck, u32 &g, u32 &info, u64 nck, u32 ng, u32 ninfo) {
  u64 e0 = ck, e1 = ((u64)info << 32) | g;
  u64 d0 = nck, d1 = ((u64)ninfo << 32) | ng;
  u64 r0, r1;
  cas128<SM>(v, e0, e1, d0, d1, r0, r1);
  bool ok = (r0 == e0) && (r1 == e1);
  ck = r0;
  g = (u32)r1;
  info = (u32)(r1 >> 32);
  return ok;
}

// A state's degree codes (record-word bits >> 27: ecode | xcode << 3) from
// the degree array, for the utterance-start token (every other state gets
// them from the arc record that reaches it).
__device__ __forceinline__ u32 state_codes(const DecodeParams &P, u32 s) {
  const u32 dg = __ldg(&P.deg[s]);
  const u32 e = dg & 15u, x = dg >> 4;
  return (e == DEG_OVF ? ECODE_OVF : e) | ((x == DEG_OVF ? XCODE_OVF : x) << 3);
}

// L2 prefetch: memory-level parallelism that costs no registers
__device__ __forceinline__ void prefetch_l2(const void *p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Bulk asynchronous copy global -> shared (the TMA engine's non-tensor mode,
// SASS UBLKCP) completing on an mbarrier: the next frame's score row lands in
// shared memory while the current frame finishes, with no thread involved.
__device__ __forceinline__ u32 smem_u32(const void *p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64 *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_row_load(void *dst, const void *src, u32 bytes, u64 *bar) {
  // the buffer's previous contents were read through the generic proxy
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64 *bar, u32 phase) {
  asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
               " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
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

// Exclusive scan of Q values per thread in q-major order (element (q, t) at
// position q * BLOCK + t): the order of coalesced loads i = base + q * BLOCK +
// tid.  One barrier: every warp scans the warp totals itself; consecutive
// calls alternate between two scratch halves (par), so a warp that is ahead
// never overwrites totals a slower warp is still reading (a barrier separates
// a call from the one two calls later).  sh needs 2 * 32 words.
template <int BLOCK, int Q>
__device__ __forceinline__ void block_excl_scan_q(const u32 (&v)[Q], u32 (&ex)[Q], u32 &total, u32 *sh, u32 par) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int NW = BLOCK / 32;
  static_assert(Q * NW <= 32, "scan scratch");
  u32 *t = sh + (par & 1u) * 32u;
  u32 x[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    x[q] = v[q];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, x[q], o);
      if (lane >= o) x[q] += y;
    }
    if (lane == 31) t[q * NW + wid] = x[q];
  }
  __syncthreads();
  u32 w = lane < Q * NW ? t[lane] : 0u;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 y = __shfl_up_sync(0xffffffffu, w, o);
    if (lane >= o) w += y;
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int k = q * NW + wid;
    const u32 before = __shfl_sync(0xffffffffu, w, (k + 31) & 31); // inclusive prefix of k - 1
    ex[q] = (k ? before : 0u) + x[q] - v[q];
  }
  total = __shfl_sync(0xffffffffu, w, Q * NW - 1);
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

// Reservation of n consecutive entries on a shared counter, aggregated over
// the lanes that are converged here (one shared atomic per group): the
// entries of a warp are contiguous, so its stores to them coalesce.
__device__ __forceinline__ u32 agg_reserve(u32 *counter, u32 n) {
  // one request per lane (the usual case): ballot + popc, one atomic per warp
  // (the cooperative-groups path below finds lanes in software)
  const u32 act = __activemask();
  if (__all_sync(act, n <= 1u)) {
    const u32 m = __ballot_sync(act, n != 0);
    if (!m) return 0;
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    u32 base = 0;
    if (lane == leader) base = atomicAdd(counter, (u32)__popc(m));
    base = __shfl_sync(act, base, leader);
    return base + (u32)__popc(m & ((1u << lane) - 1u));
  }
  namespace cg = cooperative_groups;
  cg::coalesced_group grp = cg::coalesced_threads();
  const u32 excl = cg::exclusive_scan(grp, n, cg::plus<u32>());
  const u32 total = grp.shfl(excl + n, grp.size() - 1);
  u32 base = 0;
  if (grp.thread_rank() == 0 && total) base = atomicAdd(counter, total);
  return grp.shfl(base, 0) + excl;
}

// agg_reserve of two counters packed in one 64-bit word (low, high halves):
// one atomic per group for both (a cluster's counters are a peer's shared
// memory, where every atomic is a round trip).
__device__ __forceinline__ void agg_reserve2(unsigned long long *counter, u32 n_lo, u32 n_hi, u32 &base_lo,
                                             u32 &base_hi) {
  const u32 act = __activemask();
  const int lane = threadIdx.x & 31;
  if (__all_sync(act, n_lo <= 1u && n_hi <= 1u)) {
    const u32 ml = __ballot_sync(act, n_lo != 0), mh = __ballot_sync(act, n_hi != 0);
    const u32 m = ml | mh;
    if (!m) {
      base_lo = base_hi = 0;
      return;
    }
    const int leader = __ffs(m) - 1;
    unsigned long long b = 0;
    if (lane == leader) b = atomicAdd(counter, (unsigned long long)__popc(ml) | ((unsigned long long)__popc(mh) << 32));
    b = __shfl_sync(act, b, leader);
    const u32 lt = (1u << lane) - 1u;
    base_lo = (u32)b + (u32)__popc(ml & lt);
    base_hi = (u32)(b >> 32) + (u32)__popc(mh & lt);
    return;
  }
  namespace cg = cooperative_groups;
  cg::coalesced_group grp = cg::coalesced_threads();
  const u32 el = cg::exclusive_scan(grp, n_lo, cg::plus<u32>());
  const u32 eh = cg::exclusive_scan(grp, n_hi, cg::plus<u32>());
  const u32 tl = grp.shfl(el + n_lo, grp.size() - 1), th = grp.shfl(eh + n_hi, grp.size() - 1);
  unsigned long long b = 0;
  if (grp.thread_rank() == 0 && (tl | th)) b = atomicAdd(counter, (unsigned long long)tl | ((unsigned long long)th << 32));
  b = grp.shfl(b, 0);
  base_lo = (u32)b + el;
  base_hi = (u32)(b >> 32) + eh;
}

// warp-aggregated append to a shared counter: one smem atomic per warp.
// Must be reached by every lane of the warp (pred may differ).
__device__ __forceinline__ u32 warp_append(u32 *counter, bool pred) {
  const u32 m = __ballot_sync(0xffffffffu, pred);
  const int lane = threadIdx.x & 31;
  u32 base = 0;
  if (m) {
    const int leader = __ffs(m) - 1;
    if (lane == leader) base = atomicAdd(counter, (u32)__popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
  }
  return base + __popc(m & ((1u << lane) - 1u));
}

// ------------------------------------------------------------ phase profile
// Built with -DAB_PROFILE only (scripts/, never the shipped library): thread 0
// accumulates SM clock cycles per phase; the kernel adds them to P.prof.
enum { PF_START = 0, PF_ROW, PF_EMIT_X, PF_EMIT_S, PF_EPS_X, PF_EPS_S, PF_PRUNE_SCAN, PF_PRUNE_SEL,
       PF_PRUNE_OUT, PF_HYP, PF_GC, PF_ROUNDS, PF_EPOCH, PF_EMIT_BAR, PF_EPS_BAR, PF_ADV_BAR, PF_WALK, PF_NHYP, PF_XLIST, PF_XCAND, PF_XRELAX, PF_PHIST, PF_PROWS, PF_NSEL, PF_NMEM, PF_NPASS, PF_N = 26 };
#ifdef AB_PROFILE
#define PROF_MARK(sh, id)                                                                          \
  do {                                                                                             \
    if (threadIdx.x == 0) {                                                                        \
      const long long t_ = clock64();                                                              \
      (sh).prof[id] += (unsigned long long)(t_ - (sh).prof_t);                                     \
      (sh).prof_t = t_;                                                                            \
    }                                                                                              \
  } while (0)
#define PROF_COUNT(sh, id, v)                                                                      \
  do {                                                                                             \
    if (threadIdx.x == 0) (sh).prof[id] += (v);                                                    \
  } while (0)
#else
#define PROF_MARK(sh, id) do { } while (0)
#define PROF_COUNT(sh, id, v) do { } while (0)
#endif

// ------------------------------------------------------------ CTA state

enum {
  E_NONE = 0,
  E_DEAD = AB_ERR_DEAD,
  E_STATUS = AB_ERR_STATUS,
  E_CAP = AB_ERR_CAPACITY
};

// A channel's counters.  With one CTA per channel they are in its shared
// memory; a channel decoded by a thread-block cluster (Fmt::cluster > 1, C1 /
// C2) keeps them in the leader CTA's, reached over DSMEM (GC()).
struct Counters {
  // n_app / n_cand: per pass, by pass index mod 3 (every thread tracks it):
  // a pass's slot is read after the pass's barrier and the slot of the pass
  // after next reset then, so a pass needs one (cluster) barrier
  // frontier rows so far | epsilon-frontier entries so far (eps_n), in one
  // 64-bit word: a warp reserves both with one atomic (agg_reserve2)
  union {
    struct {
      u32 flog_n, eps_n;
    };
    unsigned long long fe_n;
  };
  u32 n_new, n_app[3], n_cand[3], rec_n;
  unsigned long long rec_logical;
  unsigned long long min_ck; // cheapest application of the current frame
  int error;
  int max_depth;
  unsigned long long cnt_tok, cnt_emit, cnt_eps;
  int n_rec_frame; // emission records of the frame (olabel != 0 applications)
  int best_last_il;
  double cut_fail; // a failed attempt's own cutoff (the next attempt's hint)
  union { // cluster prune: survivors | split-bucket rows reserved so far (one atomic reserves both)
    struct {
      u32 out_tok, out_mem;
    };
    unsigned long long out_tm;
  };
  u32 out_sel;          // cluster prune: survivors after the split-bucket selection
};

// A partial hypothesis picked but not yet walked (cluster: deferred to the
// next frame's emitting pass, see emit_pending_warp).
struct PendHyp {
  double cost;
  long long frame;
  int out_idx, bp, depth, hits;
};

struct Shared {
  Counters cnt;    // this channel's counters (leader CTA of a cluster)
  u32 emit_end;    // rows below come from the emitting pass (their source is a token); every CTA's copy
  u32 pe_row0, pe_n_cand, pe_n_app, pe_eps_n; // pass_end_c: the leader's counts, read once per CTA
  int pe_error;
  PendHyp pend;    // (leader CTA) the deferred partial hypothesis
  Counters *lead;  // the leader's counters (cluster mode: a DSMEM address)
  u32 sel;
  u32 cum;
  u32 out_base_tok, out_base_mem; // cluster prune: a tile's reserved output positions
  u64 xbest_k; // cluster prune: this CTA's best (cost, state) row, read by its peers
  u32 xbest_s;
  int xbest_i;
  int shared_words;
  long long words_off;
  // scan / reduce scratch
  u32 scan[64]; // (block_excl_scan_q: two halves)
  u64 redk[32];
  u32 reds[32];
  int redi[32];
  // live rows of the frame by cost bucket, kept while rows are written and
  // killed (prune finds its split bucket without a pass over the rows)
  u32 fhist[1024];
  double hbase, hscale;
  double cut_hint; // this attempt's cutoff hint (inf: unfiltered), see advance()
  int filtered;
  // next frame's score row, bulk-copied into the row buffer once the current
  // frame's emitting pass is final (prune verified it; see decode_kernel)
  const void *next_row;
  u64 row_bar;
  u32 row_phase;
  int row_pending;
#ifdef AB_PROFILE
  unsigned long long prof[PF_N];
  long long prof_t;
#endif
};

// The channel's counters: this CTA's, or the cluster leader's (DSMEM).
template <typename F> __device__ __forceinline__ Counters &GC(Shared &sh) {
  if constexpr (F::cluster > 1) return *sh.lead;
  else return sh.cnt;
}

// Rank of this CTA in the channel's cluster (0 = leader) and the channel-wide
// barrier: the cluster barrier (release / acquire at cluster scope, so the
// leader's counters and every CTA's global writes are visible after it) or
// the CTA barrier.
template <typename F> __device__ __forceinline__ u32 crank() {
  if constexpr (F::cluster > 1) {
    u32 r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
  } else {
    return 0;
  }
}
template <typename F> __device__ __forceinline__ void csync() {
  if constexpr (F::cluster > 1)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else
    __syncthreads();
}
// thread 0 of the channel (the leader CTA's)
template <typename F> __device__ __forceinline__ bool chan_t0() { return threadIdx.x == 0 && crank<F>() == 0; }

template <typename F, typename S> struct Chan {
  const DecodeParams *P;
  int b; // batch index of the channel this CTA is decoding
  int slot;
  ChanState *cs;
  Entry *table;
  u64 *vals;
  u64 *gvals; // the channel's global direct table (wiped with a shared-memory table)
  double prev_best, prev_cut, cut_rise; // this CTA's copy of ChanState's (every CTA updates it alike)
  u64 *peer_vals[F::cluster]; // cluster: every CTA's part of the shared-memory table (generic DSMEM addresses)
  Shared *peer_sh[F::cluster]; // cluster: every CTA's Shared (histograms, per-CTA best tokens)
  u32 *tok_state;
  double *tok_cost;
  TokInfo *tok_info;
  u32 *flog_state;
  u64 *flog_ck;
  uint4 *flog_aux;
  uint4 *eps_list;
  TokInfo *tok_info_alt; // the other half of the channel's provenance buffer
  u32 *app_list;
  u32 *kill; // the channel's kill words (KW_*)
  u64 *scr_key;
  u32 *scr_row;
  int2 *arena; // live half
  int2 *arena_to;
  u32 *gc_bits;
  u32 *gc_rank;
  int *path_rec;
  int *path_words;
  const S *row;
  // context
  double discount;
  int ctx_mode;
  const u32 *ctx_list; // hash set of the context's arc ids
  u32 ctx_k, ctx_lmask;
  const u32 *ctx_bits;
  const u32 *ctx_bits_x;
  u32 ctx_words;
  u32 epoch;
  u32 etag;
  double slack; // the context's epsilon slack (CtxDesc::slack)
  int slack_rounds;
  double ucut0; // this attempt's candidate cutoff (candidates above it are not relaxed) ...
  double ucut;  // ... plus the slack, for states in the slack Bloom filter
  const u32 *neg; // shared-memory copy of the context's (or graph's) slack Bloom filter
  u32 neg_fold; // log2(NEG_WORDS / the launch's filter words)
  const u32 *hq; // or the context's per-state 2-bit slack (CtxDesc::hq)
  const u32 *fbits, *fbits_x; // (with hq) records whose destination has a slack, by position
  double hq_unit;
  // expansion tile (shared memory)
  u32 *t_a0;
  u32 *t_pref;
  u32 *t_src;
  double *t_cost;
  u32 *t_coarse; // CTA tiles: owner of every 32nd arc (TILE_COARSE entries)
};

// The cheapest application of the frame: this CTA's, or the minimum over the
// cluster's CTAs (each keeps its own, see expand).
template <typename F, typename S> __device__ __forceinline__ u64 frame_min_ck(const Chan<F, S> &C, Shared &sh) {
  if constexpr (F::cluster > 1) {
    u64 m = ~0ull;
#pragma unroll
    for (int r = 0; r < F::cluster; ++r) m = min(m, C.peer_sh[r]->cnt.min_ck);
    return m;
  } else {
    return sh.cnt.min_ck;
  }
}

constexpr u32 NB_HIST = 1024;
constexpr double HIST_PER_BEAM = 256.0; // buckets per beam width
// Cost bucket of the frame's histogram: monotone in the cost, clamped at both ends.
__device__ __forceinline__ u32 hbucket(const Shared &sh, double c) {
  const double x = (c - sh.hbase) * sh.hscale;
  // !(x > 0) also catches NaN (an infinite beam makes the scale 0 and the base -inf)
  return !(x > 0.0) ? 0u : (x >= (double)(NB_HIST - 1) ? NB_HIST - 1 : (u32)x);
}

// Bitset word of a BITSET context for the arc record at position a: addressed
// by position, so it is loaded next to the record, not after it.
template <bool EMIT, typename F, typename S>
__device__ __forceinline__ u32 boost_word(const Chan<F, S> &C, u32 a) {
  return C.ctx_mode == CTX_BITSET ? __ldg(&(EMIT ? C.ctx_bits : C.ctx_bits_x)[a >> 5]) : 0u;
}
// Slack-flag word of a dense context for the record at position a (ditto).
template <bool EMIT, typename F, typename S>
__device__ __forceinline__ u32 slack_word(const Chan<F, S> &C, u32 a) {
  return C.hq ? __ldg(&(EMIT ? C.fbits : C.fbits_x)[a >> 5]) : 0u;
}

// BiasingContext.boosted_mask (biasing.py:108-117) in the representation the
// context store chose for this context; bw = boost_word of the record.
template <typename F, typename S>
__device__ __forceinline__ bool is_boosted(const Chan<F, S> &C, u32 a, u32 bw, u32 g, u32 ol) {
  switch (C.ctx_mode) {
  case CTX_NONE: return false;
  case CTX_LABELS: return ol < C.ctx_words * 32u && ((C.ctx_bits[ol >> 5] >> (ol & 31)) & 1u);
  case CTX_BITSET: return (bw >> (a & 31)) & 1u;
  case CTX_SLIST: { // Bloom filter (shared), then the id set (global) for its few hits
    const u32 nb = C.ctx_words * 32u, b1 = list_b1(g, nb), b2 = list_b2(g, nb);
    if (!((C.ctx_bits[b1 >> 5] >> (b1 & 31)) & (C.ctx_bits[b2 >> 5] >> (b2 & 31)) & 1u)) return false;
  } // fall through
  default: {
    // CTX_GLIST (and the filter's hits): the hash set in global memory
    if (C.ctx_k == 0) return false;
    const u32 *a = C.ctx_list;
    for (u32 h = list_slot(g, C.ctx_lmask);; h = (h + 1) & C.ctx_lmask) {
      const u32 v = __ldg(a + h);
      if (v == g) return true;
      if (v == 0xFFFFFFFFu) return false;
    }
  }
  }
}

// One candidate: cost in the reference's association order with the boost
// fused into the weight (_effective_weights, decoder.py:234-240, 378 emitting,
// 268 epsilon), its row flags, and whether it is relaxed at all: a candidate
// above the frame's cutoff is provably outside the survivors (advance(); a
// destination without epsilon arcs has no epsilon path, hence no slack).
template <bool EMIT, typename F, typename S>
__device__ __forceinline__ bool candidate(const Chan<F, S> &C, double cj, double w, u32 il, u32 ol, u32 g, u32 d,
                                          u32 a, u32 bw, u32 fw, u64 &ck, u32 &rflags) {
  const bool bst = is_boosted(C, a, bw, g & G_MASK, ol);
  const double we = bst ? w + C.discount : w;
  const double cand = EMIT ? (cj + we) + (double)C.row[il - 1] : cj + we;
  ck = cost_key(cand);
  rflags = (bst ? ROW_BOOST : 0u) | (ol ? ROW_HASOL : 0u) | ((g & G_DEST_EPS) ? ROW_EPS : 0u);
  if (cand <= C.ucut0) return true;
  if (!(cand <= C.ucut) || !(g & G_DEST_EPS)) return false;
  if (C.hq) {
    if (!((fw >> (a & 31u)) & 1u)) return false; // no slack at this destination
    const u32 q = (__ldg(C.hq + d / HQ_PER_WORD) >> ((d % HQ_PER_WORD) * HQ_BITS)) & HQ_MAX;
    return q && cand <= C.ucut0 + (double)q * C.hq_unit;
  }
  return neg_test(C.neg, d, C.neg_fold);
}

template <typename F> __device__ __forceinline__ void set_error(Shared &sh, int code) {
  atomicCAS(&GC<F>(sh).error, 0, code);
}

template <bool H> __device__ __forceinline__ u32 home_slot(const DecodeParams &P, u32 d) {
  return H ? ((d * 2654435761u) >> P.hash_shift) & P.table_mask : d;
}
// value of a slot
template <typename F, typename S> __device__ __forceinline__ u64 *val_at(const Chan<F, S> &C, u32 slot) {
  // a cluster's table: state s in CTA s % cluster, at s / cluster
  if constexpr (F::cluster > 1) return C.peer_vals[slot % F::cluster] + 2 * (size_t)(slot / F::cluster);
  return F::hashed ? &C.table[slot].ck : C.vals + 2 * (size_t)slot;
}

// Relaxation (decoder.py:213-220 emitting, 277-308 epsilon) is a CAS-128
// minimum on the slot's value with the phase rule
//   empty (stale tag)           -> take it: a new token of this frame
//   value from an earlier round -> replace iff strictly cheaper (cost only)
//   value from this round       -> replace iff (cost, arc) is smaller
// A candidate that passes the check against the loaded value first writes its
// frontier row {state | flags, cost key, (source, arc id)} at a freshly
// reserved index, then installs (cost, arc, round | tag | row) by CAS.  The
// value therefore always names the row of the slot's current winner; a CAS
// that replaces a winner of the same round marks that row displaced (not an
// application), one that replaces an earlier round's winner marks it
// superseded (an application, no longer a token), in the row's kill word, so
// the rows of a round are final at the round's barrier without a second pass
// over the table.
__device__ __forceinline__ bool value_better(u64 ck, u32 g, u32 row0, u32 etag, u64 vck, u32 vg,
                                             u32 vinfo) {
  const bool valid = ((vinfo >> TAG_SHIFT) & TAG_MASK) == etag;
  const bool earlier = (vinfo & VROW_MASK) < row0; // installed in an earlier round of the frame
  return !valid || (earlier ? (ck < vck) : (ck < vck || (ck == vck && g < vg)));
}

struct RelaxAcc {
  u64 min_ck;  // cheapest installed candidate
  u32 n_new;   // new tokens (capacity check)
  u32 n_app;   // applications (decoder.py:285-287 stop rule)
  int n_rec;   // rows written with an output label (emission records, net of self-displacement)
};

// DEAD / DISP of a cluster's row (0 if neither), from its kill word.
template <typename F, typename S> __device__ __forceinline__ u32 kill_flags(const Chan<F, S> &C, u32 row) {
  const u32 w = C.kill[row];
  return (w >> 2) != C.etag ? 0u : (w & KW_DEAD) ? ROW_DEAD : ROW_DISP;
}

// Outcome of a successful CAS that replaced old_info.
template <typename F, typename S>
__device__ __forceinline__ void installed(const DecodeParams &P, const Chan<F, S> &C, Shared &sh, RelaxAcc &acc,
                                          u32 row0, u32 etag, u32 old_info, u64 old_ck, u64 ck) {
  acc.min_ck = min(acc.min_ck, ck);
  if (((old_info >> TAG_SHIFT) & TAG_MASK) != etag) {
    acc.n_new++;
    acc.n_app++;
    return;
  }
  // the replaced winner's row leaves the live rows (its cost is the CAS's expected key)
  atomicSub(&sh.fhist[hbucket(sh, key_cost(old_ck))], 1u);
  const bool earlier = (old_info & VROW_MASK) < row0;
  acc.n_app += earlier ? 1 : 0;
  C.kill[old_info & VROW_MASK] = (etag << 2) | (earlier ? KW_DEAD : KW_DISP);
}

// CAS retry loop after a lost race; the candidate's row is `row`.  A
// candidate that stops being better marks its own row displaced.
template <typename F, typename S>
__device__ void relax_retry(const DecodeParams &P, const Chan<F, S> &C, Shared &sh, RelaxAcc &acc, u64 *v,
                            u64 ck, u32 g, u32 info, u32 row0, u64 vck, u32 vg, u32 vinfo, u32 row,
                            bool hasol) {
  const u32 etag = C.etag;
  while (true) {
    if (!value_better(ck, g, row0, etag, vck, vg, vinfo)) {
      C.kill[row] = (etag << 2) | KW_DISP;
      atomicSub(&sh.fhist[hbucket(sh, key_cost(ck))], 1u);
      acc.n_rec -= hasol ? 1 : 0;
      return;
    }
    const u32 old_info = vinfo;
    const u64 old_ck = vck;
    if (cas_value<table_space<F>()>(v, vck, vg, vinfo, ck, g, info)) {
      installed(P, C, sh, acc, row0, etag, old_info, old_ck, ck);
      return;
    }
  }
}

// Sequential relaxation with linear probing (hashed tables: the home slot
// belongs to another state).  (key, vck, vg, vinfo) = contents of `slot`.
template <typename F, typename S>
__device__ __noinline__ void relax_probe(const DecodeParams &P, const Chan<F, S> &C, Shared &sh, RelaxAcc &acc,
                                         u32 d, u32 dc, u64 ck, u32 g, u32 src, u32 rflags, u32 lab_ol, u32 lab_il,
                                         u32 row0, u32 slot, u64 key, u64 vck, u32 vg, u32 vinfo) {
  const u64 ep = (u64)C.epoch << 32;
  u32 probes = 0;
  while (true) {
    Entry *e = &C.table[slot];
    if ((key & KEY_EPOCH_MASK) != ep) {
      const u64 want = (u64)d | ep;
      const u64 old = atomicCAS(&e->key, key, want);
      key = old == key ? want : old;
      continue;
    }
    if ((u32)key == d) break;
    slot = (slot + 1) & P.table_mask;
    if (++probes > P.table_mask) {
      set_error<F>(sh, E_CAP);
      return;
    }
    ld_cg_entry(&C.table[slot], key, vck, vg, vinfo);
  }
  if (!value_better(ck, g, row0, C.etag, vck, vg, vinfo)) return;
  const u32 row = (u32)atomicAdd(&GC<F>(sh).fe_n, 1ull);
  if (row >= P.flog_cap) {
    set_error<F>(sh, E_CAP);
    return;
  }
  C.flog_state[row] = d | (ecode_of(dc) << CODE_SHIFT);
  C.flog_ck[row] = ck;
  if (rflags & ROW_EPS) {
    const u32 epos = (u32)(atomicAdd(&GC<F>(sh).fe_n, 1ull << 32) >> 32);
    C.eps_list[epos] = make_uint4(row, d | (xcode_of(dc) << CODE_SHIFT), (u32)ck, (u32)(ck >> 32));
  }
  store_aux<1024, F>(C.flog_aux, row, aux_src(src, rflags, g), lab_ol, lab_il);
  atomicAdd(&sh.fhist[hbucket(sh, key_cost(ck))], 1u);
  acc.n_rec += (rflags & ROW_HASOL) ? 1 : 0;
  const u32 info = (C.etag << TAG_SHIFT) | row;
  relax_retry(P, C, sh, acc, val_at(C, slot), ck, g, info, row0, vck, vg, vinfo, row,
              (rflags & ROW_HASOL) != 0);
}

// Relaxation of U independent candidates of one thread.  Every memory step
// is issued for all U candidates before any result is consumed: loads of the
// slots, key claims (hashed tables), row writes, value CAS-128s.  Lost races
// and probe chains fall back to the sequential path.
template <int BLOCK, int U, typename F, typename S>
__device__ __forceinline__ void relax_batch(const DecodeParams &P, const Chan<F, S> &C, Shared &sh, RelaxAcc &acc,
                                            const bool (&on)[U], const u32 (&d)[U], const u32 (&dc)[U],
                                            const u64 (&ck)[U],
                                            const u32 (&g)[U], const u32 (&src)[U], const u32 (&rflags)[U],
                                            const u32 (&ol)[U], const u32 (&il)[U], u32 row0) {
  const u32 etag = C.etag;
  const u64 ep = (u64)C.epoch << 32;
  u32 slot[U];
  u64 key[U], vck[U];
  u32 vg[U], vinfo[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    slot[u] = home_slot<F::hashed>(P, d[u]);
    key[u] = 0;
    vck[u] = 0;
    vg[u] = 0;
    vinfo[u] = 0;
    if (on[u]) {
      if (F::hashed) ld_cg_entry(&C.table[slot[u]], key[u], vck[u], vg[u], vinfo[u]);
      else ld_cg_value<table_space<F>()>(val_at(C, slot[u]), vck[u], vg[u], vinfo[u]);
    }
  }
  bool fast[U];
  if (F::hashed) {
    u64 old[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (on[u] && (key[u] & KEY_EPOCH_MASK) != ep)
        old[u] = atomicCAS(&C.table[slot[u]].key, key[u], (u64)d[u] | ep);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (on[u] && (key[u] & KEY_EPOCH_MASK) != ep) key[u] = old[u] == key[u] ? ((u64)d[u] | ep) : old[u];
      fast[u] = on[u] && (key[u] & KEY_EPOCH_MASK) == ep && (u32)key[u] == d[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (on[u] && !fast[u])
        relax_probe<F, S>(P, C, sh, acc, d[u], dc[u], ck[u], g[u], src[u], rflags[u], ol[u], il[u], row0,
                          slot[u], key[u], vck[u], vg[u], vinfo[u]);
  } else {
#pragma unroll
    for (int u = 0; u < U; ++u) fast[u] = on[u];
  }
  bool want[U];
  u32 nw = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    want[u] = fast[u] && value_better(ck[u], g[u], row0, etag, vck[u], vg[u], vinfo[u]);
    nw += want[u] ? 1u : 0u;
  }
  if (!nw) return;
  u32 ne = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) ne += (want[u] && (rflags[u] & ROW_EPS)) ? 1u : 0u;
  u32 row, ep_at;
  agg_reserve2(&GC<F>(sh).fe_n, nw, ne, row, ep_at);
  if (row + nw > P.flog_cap) {
    set_error<F>(sh, E_CAP);
    return;
  }
  u32 rows[U], ninfo[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    rows[u] = 0;
    ninfo[u] = 0;
    if (!want[u]) continue;
    rows[u] = row++;
    if (rflags[u] & ROW_EPS) { // next round's epsilon frontier
      st_row<BLOCK>(&C.eps_list[ep_at++],
                    make_uint4(rows[u], d[u] | (xcode_of(dc[u]) << CODE_SHIFT), (u32)ck[u], (u32)(ck[u] >> 32)));
    }
    st_row<BLOCK>(&C.flog_state[rows[u]], d[u] | (ecode_of(dc[u]) << CODE_SHIFT) |
                                              ((rflags[u] & ROW_HASOL) ? ROW_REC : 0u));
    st_row<BLOCK>(&C.flog_ck[rows[u]], (unsigned long long)ck[u]);
    store_aux<BLOCK, F>(C.flog_aux, rows[u], aux_src(src[u], rflags[u], g[u]), ol[u], il[u]);
    atomicAdd(&sh.fhist[hbucket(sh, key_cost(ck[u]))], 1u);
    acc.n_rec += (rflags[u] & ROW_HASOL) ? 1 : 0;
    ninfo[u] = (etag << TAG_SHIFT) | rows[u];
  }
  u64 r0[U], r1[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (want[u])
      cas128<table_space<F>()>(val_at(C, slot[u]), vck[u], ((u64)vinfo[u] << 32) | vg[u], ck[u], ((u64)ninfo[u] << 32) | g[u],
             r0[u], r1[u]);
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (!want[u]) continue;
    if (r0[u] == vck[u] && r1[u] == (((u64)vinfo[u] << 32) | vg[u]))
      installed(P, C, sh, acc, row0, etag, vinfo[u], vck[u], ck[u]);
    else
      relax_retry(P, C, sh, acc, val_at(C, slot[u]), ck[u], g[u], ninfo[u], row0, r0[u], (u32)r1[u],
                  (u32)(r1[u] >> 32), rows[u], (rflags[u] & ROW_HASOL) != 0);
  }
}

// Expansion of an input list over one CSR, in tiles of BLOCK * Q inputs:
// the emitting pass expands the token list (source = token index), an
// epsilon round the frontier rows listed in `list` (rows of the previous round
// whose state has epsilon arcs, appended when they were written; displaced
// ones are skipped; source = row index).
//   1. each thread loads Q consecutive inputs and their CSR ranges (all loads
//      independent), one block scan of the out-degrees;
//   2. arcs k = tid, tid + BLOCK, ... (warp-coalesced arc records), U per
//      thread in flight: arc-record loads, candidates (boost lookup fused
//      into the cost add), one batched relaxation.
template <int BLOCK, int Q, int U, bool EMIT, typename F, typename S>
__device__ void expand(const DecodeParams &P, const Chan<F, S> &C, Shared &sh, const uint4 *list, u32 n_in,
                       u32 row0, u32 slot, bool skip0 = false) {
  constexpr u32 TILE = BLOCK * Q;
  // 1024-thread CTAs (one channel alone on its SM, C1 / C2): warp-private
  // sub-tiles, no CTA barrier inside the pass; smaller CTAs share their SM
  // with other channels, which hide the tile barrier (CTA-wide tiles)
  constexpr bool WARP_TILES = AB_WARP_TILES_MIN_BLOCK > 0 && BLOCK >= AB_WARP_TILES_MIN_BLOCK;
  u32 *t_a0 = C.t_a0;
  u32 *t_pref = C.t_pref;
  u32 *t_src = C.t_src;
  double *t_cost = C.t_cost;
  const int tid = threadIdx.x;
  const uint2 *rng = EMIT ? P.e_rng : P.x_rng;
  constexpr u32 SLOT = EMIT ? SLOT_E : SLOT_X;
  const void *arcs = EMIT ? P.e_arcs : P.x_arcs;
  RelaxAcc acc;
  acc.min_ck = ~0ull;
  acc.n_new = 0;
  acc.n_app = 0;
  acc.n_rec = 0;
  u32 arcs_seen = 0;
  if constexpr (WARP_TILES) {
  // Each warp works through its own sub-tiles (32 * Q inputs; smaller when
  // the input is short, so every warp gets some): a warp-level scan of the
  // out-degrees, then its 32 lanes walk the sub-tile's arcs.  No block
  // barrier inside the pass, so a warp never waits for the slowest warp of
  // the CTA between tiles.
  constexpr u32 NW = BLOCK / 32;
  constexpr u32 WT = 32 * Q;
  const u32 lane = (u32)tid & 31u, wid = (u32)tid >> 5;
  u32 *w_a0 = t_a0 + wid * WT;
  u32 *w_pref = t_pref + wid * WT;
  u32 *w_src = t_src + wid * WT;
  double *w_cost = t_cost + wid * WT;
  // a cluster's warps share the inputs: warp (rank, wid) is global warp gw of CL * NW
  // (skip0: the cluster's warp 0 is busy elsewhere, the others share the inputs)
  const u32 GW = NW * F::cluster - (skip0 ? 1u : 0u);
  const u32 gw0 = crank<F>() * NW + wid;
  const u32 gw = skip0 ? gw0 - 1u : gw0;
  const u32 per = n_in >= GW * WT ? WT : max(1u, (n_in + GW - 1) / GW);
  for (u32 base = gw * per; base < n_in && !(skip0 && gw0 == 0); base += GW * per) {
    const u32 ne = min(per, n_in - base);
    u32 idx[Q], st[Q], a0[Q], cnt[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const u32 j = lane * Q + q;
      idx[q] = 0xFFFFFFFFu;
      st[q] = ROW_DISP;
      if (j < ne) {
        if (EMIT) {
          idx[q] = base + j;
          st[q] = C.tok_state[idx[q]];
          w_cost[j] = C.tok_cost[idx[q]];
        } else { // epsilon-frontier entries carry the row's state, flags and cost
          const uint4 e = list[base + j];
          idx[q] = e.x;
          st[q] = e.y | (kill_flags(C, e.x) & ROW_DISP); // displaced after listing
          w_cost[j] = key_cost(((u64)e.w << 32) | e.z);
        }
        w_src[j] = idx[q];
      }
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      a0[q] = 0;
      cnt[q] = 0;
      // (with the DISP check at listing, the degree load does not wait for it)
      if (idx[q] != 0xFFFFFFFFu) {
        const u32 s = st[q] & ROW_STATE;
        const u32 c = EMIT ? (st[q] >> CODE_SHIFT) & 7u : (st[q] >> CODE_SHIFT) & 3u;
        if (c == (EMIT ? ECODE_OVF : XCODE_OVF)) {
          const uint2 r = __ldg(&rng[s]);
          a0[q] = r.x;
          cnt[q] = r.y - r.x;
        } else {
          a0[q] = s * SLOT;
          cnt[q] = c;
        }
        if (!EMIT && (st[q] & ROW_DISP)) cnt[q] = 0; // displaced: not expanded
      }
    }
    u32 tsum = 0;
#pragma unroll
    for (int q = 0; q < Q; ++q) tsum += cnt[q];
    u32 incl = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= (u32)o) incl += y;
    }
    const u32 total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    PROF_MARK(sh, PF_XLIST);
    u32 run = incl - tsum;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const u32 j = lane * Q + q;
      if (j < ne) {
        w_a0[j] = a0[q];
        w_pref[j] = run;
      }
      run += cnt[q];
    }
    __syncwarp();
    arcs_seen += total;
    for (u32 k0 = lane; k0 < total; k0 += 32 * U) {
      bool on[U];
      u32 a[U], src[U];
      double cj[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const u32 k = k0 + u * 32;
        on[u] = k < total;
        a[u] = 0;
        src[u] = 0;
        cj[u] = 0.0;
        if (on[u]) {
          u32 lo = 0, hi = ne - 1; // largest j with w_pref[j] <= k (its range holds k)
          while (lo < hi) {
            const u32 mid = (lo + hi + 1) >> 1;
            if (w_pref[mid] <= k) lo = mid;
            else hi = mid - 1;
          }
          a[u] = w_a0[lo] + (k - w_pref[lo]);
          src[u] = w_src[lo];
          cj[u] = w_cost[lo];
        }
      }
      u32 d[U], dc[U], g[U], il[U], ol[U], bw[U], fw[U];
      double w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        d[u] = g[u] = il[u] = ol[u] = 0;
        w[u] = 0.0;
        bw[u] = 0;
        fw[u] = 0;
        if (on[u]) {
          bw[u] = boost_word<EMIT>(C, a[u]);
          fw[u] = slack_word<EMIT>(C, a[u]);
          if (EMIT) F::emit(arcs, a[u], d[u], g[u], w[u], il[u], ol[u]);
          else F::eps(arcs, a[u], d[u], g[u], w[u], ol[u]);
        }
        dc[u] = d[u] >> CODE_SHIFT; // the destination's degree codes
        d[u] &= ROW_STATE;
      }
      u64 ck[U];
      u32 rflags[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        ck[u] = 0;
        rflags[u] = 0;
        if (on[u]) on[u] = candidate<EMIT>(C, cj[u], w[u], il[u], ol[u], g[u], d[u], a[u], bw[u], fw[u], ck[u], rflags[u]);
      }
      PROF_MARK(sh, PF_XCAND);
      relax_batch<BLOCK, U>(P, C, sh, acc, on, d, dc, ck, g, src, rflags, ol, il, row0);
      PROF_MARK(sh, PF_XRELAX);
    }
    __syncwarp();
  }
  if (lane == 0 && arcs_seen) {
    atomicAdd(&GC<F>(sh).n_cand[slot], arcs_seen);
    atomicAdd(EMIT ? &GC<F>(sh).cnt_emit : &GC<F>(sh).cnt_eps, (unsigned long long)arcs_seen);
  }
  } else {
  // tile position j = q * BLOCK + tid: input base + j, so every load of the
  // tile's inputs is warp-coalesced (the degree scan runs in the same order)
  // (the tile's shared arrays are written after the degree scan, whose
  // barriers every thread reaches only after the previous tile's arcs: no
  // barrier at the end of a tile)
  for (u32 base = 0; base < n_in; base += TILE) {
    u32 idx[Q], st[Q], a0[Q], cnt[Q];
    double cq[Q];
    if (EMIT) {
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const u32 i = base + (u32)q * BLOCK + (u32)tid;
        idx[q] = i < n_in ? i : 0xFFFFFFFFu;
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) st[q] = idx[q] == 0xFFFFFFFFu ? ROW_DISP : C.tok_state[idx[q]];
#pragma unroll
      for (int q = 0; q < Q; ++q) cq[q] = idx[q] != 0xFFFFFFFFu ? C.tok_cost[idx[q]] : 0.0;
    } else {
      // epsilon-frontier entries carry the row's state, flags and cost
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const u32 j = (u32)q * BLOCK + (u32)tid;
        idx[q] = 0xFFFFFFFFu;
        st[q] = ROW_DISP;
        cq[q] = 0.0;
        if (base + j < n_in) {
          const uint4 e = list[base + j];
          idx[q] = e.x;
          st[q] = e.y | (kill_flags(C, e.x) & ROW_DISP); // displaced after listing
          cq[q] = key_cost(((u64)e.w << 32) | e.z);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      a0[q] = 0;
      cnt[q] = 0;
      // (with the DISP check at listing, the degree load does not wait for it)
      if (idx[q] != 0xFFFFFFFFu) {
        const u32 s = st[q] & ROW_STATE;
        const u32 c = EMIT ? (st[q] >> CODE_SHIFT) & 7u : (st[q] >> CODE_SHIFT) & 3u;
        if (c == (EMIT ? ECODE_OVF : XCODE_OVF)) {
          const uint2 r = __ldg(&rng[s]);
          a0[q] = r.x;
          cnt[q] = r.y - r.x;
        } else {
          a0[q] = s * SLOT;
          cnt[q] = c;
        }
        if (!EMIT && (st[q] & ROW_DISP)) cnt[q] = 0; // displaced: not expanded
      }
    }
    u32 total, pref[Q];
    block_excl_scan_q<BLOCK, Q>(cnt, pref, total, sh.scan, base / TILE);
    // coarse index of the arc -> input search: the input owning arc 32 b
    // (written by the input whose range holds it) bounds every arc of block b
    const bool coarse = total <= 32u * TILE_COARSE;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const u32 j = (u32)q * BLOCK + (u32)tid;
      t_a0[j] = a0[q];
      t_pref[j] = pref[q];
      t_src[j] = idx[q];
      t_cost[j] = cq[q];
      if (coarse)
        for (u32 m = (pref[q] + 31u) & ~31u; m < pref[q] + cnt[q]; m += 32u) C.t_coarse[m >> 5] = j;
    }
    if (tid == 0) t_pref[TILE] = total;
    __syncthreads();
    const u32 nblk = (total + 31u) >> 5;
    arcs_seen += total;
    // arcs k = tid, tid + BLOCK, ...: the lanes of a warp read consecutive
    // arc records (one state's arcs are contiguous), so a warp load touches
    // few lines; each thread keeps U such arcs in flight
    for (u32 k0 = tid; k0 < total; k0 += BLOCK * U) {
      bool on[U];
      u32 a[U], src[U];
      double cj[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const u32 k = k0 + u * BLOCK;
        on[u] = k < total;
        a[u] = 0;
        src[u] = 0;
        cj[u] = 0.0;
        if (on[u]) {
          // largest j with t_pref[j] <= k (its range holds k), between the
          // owners of the 32-arc blocks around k
          u32 lo = 0, hi = TILE - 1;
          if (coarse) {
            const u32 b = k >> 5;
            lo = C.t_coarse[b];
            if (b + 1 < nblk) hi = C.t_coarse[b + 1];
          }
          while (lo < hi) {
            const u32 mid = (lo + hi + 1) >> 1;
            if (t_pref[mid] <= k) lo = mid;
            else hi = mid - 1;
          }
          a[u] = t_a0[lo] + (k - t_pref[lo]);
          src[u] = t_src[lo];
          cj[u] = t_cost[lo];
        }
      }
      u32 d[U], dc[U], g[U], il[U], ol[U], bw[U], fw[U];
      double w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        d[u] = g[u] = il[u] = ol[u] = 0;
        w[u] = 0.0;
        bw[u] = 0;
        fw[u] = 0;
        if (on[u]) {
          bw[u] = boost_word<EMIT>(C, a[u]);
          fw[u] = slack_word<EMIT>(C, a[u]);
          if (EMIT) F::emit(arcs, a[u], d[u], g[u], w[u], il[u], ol[u]);
          else F::eps(arcs, a[u], d[u], g[u], w[u], ol[u]);
        }
        dc[u] = d[u] >> CODE_SHIFT; // the destination's degree codes
        d[u] &= ROW_STATE;
      }
      u64 ck[U];
      u32 rflags[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        ck[u] = 0;
        rflags[u] = 0;
        if (on[u]) on[u] = candidate<EMIT>(C, cj[u], w[u], il[u], ol[u], g[u], d[u], a[u], bw[u], fw[u], ck[u], rflags[u]);
      }
      relax_batch<BLOCK, U>(P, C, sh, acc, on, d, dc, ck, g, src, rflags, ol, il, row0);
    }
  }
  }
  // per-warp totals first: one shared atomic per warp and counter
  u64 mck = acc.min_ck;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mck = min(mck, __shfl_xor_sync(0xFFFFFFFFu, mck, o));
  const int n_rec = __reduce_add_sync(0xFFFFFFFFu, acc.n_rec);
  const u32 n_app = __reduce_add_sync(0xFFFFFFFFu, acc.n_app);
  const u32 n_new = __reduce_add_sync(0xFFFFFFFFu, acc.n_new);
  if ((tid & 31) == 0) {
    // (each CTA's own minimum: a 64-bit atomicMin into a peer CTA's shared
    // memory is not atomic on sm_100, bench_tools/dsmem_atomics_probe.cu)
    if (mck != ~0ull) atomicMin(&sh.cnt.min_ck, mck);
    if (n_app) atomicAdd(&GC<F>(sh).n_app[slot], n_app);
    if (n_new && atomicAdd(&GC<F>(sh).n_new, n_new) + n_new > P.tok_cap) set_error<F>(sh, E_CAP);
  }
  static_assert(F::cluster == 1 || WARP_TILES, "a cluster's channel uses warp tiles");
  if (tid == 0 && crank<F>() == 0) {
    if (EMIT) GC<F>(sh).cnt_tok += n_in; // epsilon rounds count their whole frontier (epsilon_rounds)
    if (!WARP_TILES) {
      GC<F>(sh).n_cand[slot] += arcs_seen;
      if (EMIT) GC<F>(sh).cnt_emit += arcs_seen;
      else GC<F>(sh).cnt_eps += arcs_seen;
    }
  }
}

// Provenance of a surviving frontier row (decoder.py:385-393, 289-295): one
// walk over the row's source links back to the token of the previous frame
// (rows below sh.emit_end are the emitting pass's; their source is a token
// index) or to the utterance start.  Each arc with olabel != 0 on the way
// gets an emission record; a record is written once the next older record of
// the chain is known, so the chain is walked only once.
template <typename F, typename S>
__device__ TokInfo resolve_row(const DecodeParams &P, const Chan<F, S> &C, Shared &sh, u32 row,
                               const TokInfo *prev_tok) {
  TokInfo base;
  base.bp = -1;
  base.depth = 0;
  base.hits = 0;
  base.last_il = 0;
  const u32 emit_end = sh.emit_end;
  if constexpr (F::cluster > 1) {
    // (a cluster's record counter is the leader's: one warp-aggregated
    // reservation after a counting walk, then the records on a second walk
    // over the same, now cached, aux words)
    int hits = 0, nrec = 0;
    u32 il = 0, cur = row;
    while (true) {
      u32 ax_x, ax_ol, ax_il;
      load_aux<F>(C.flog_aux, cur, ax_x, ax_ol, ax_il);
      if (ax_x & AUX_START) break;
      hits += (ax_x & AUX_BOOST) ? 1 : 0;
      nrec += (ax_x & AUX_HASOL) ? 1 : 0;
      if (cur < emit_end) {
        il = ax_il;
        base = prev_tok[ax_x & AUX_SRC];
        break;
      }
      cur = ax_x & AUX_SRC;
    }
    const u32 r0 = agg_reserve(&GC<F>(sh).rec_n, (u32)nrec);
    if (nrec && r0 + (u32)nrec > P.arena_cap) {
      set_error<F>(sh, E_CAP);
      nrec = 0;
    }
    cur = row;
    for (int j = 0; j < nrec;) {
      u32 ax_x, ax_ol, ax_il;
      load_aux<F>(C.flog_aux, cur, ax_x, ax_ol, ax_il);
      if (ax_x & AUX_HASOL) { // record r0 + j (newest first) -> the next older one
        C.arena[r0 + j] = make_int2((int)ax_ol, j + 1 < nrec ? (int)(r0 + j + 1) : base.bp);
        ++j;
      }
      cur = ax_x & AUX_SRC;
    }
    TokInfo t;
    t.hits = base.hits + hits;
    t.depth = base.depth + nrec;
    t.last_il = (int)il;
    t.bp = nrec ? (int)r0 : base.bp;
    return t;
  }
  int hits = 0, nrec = 0, newest = -1, pend = -1;
  u32 pend_ol = 0, il = 0;
  u32 cur = row;
  while (true) {
    u32 ax_x, ax_ol, ax_il;
    load_aux<F>(C.flog_aux, cur, ax_x, ax_ol, ax_il);
    if (ax_x & AUX_START) break;
    hits += (ax_x & AUX_BOOST) ? 1 : 0;
    if (ax_x & AUX_HASOL) {
      const u32 r = atomicAdd(&GC<F>(sh).rec_n, 1u);
      if (r >= P.arena_cap) {
        set_error<F>(sh, E_CAP);
        break;
      }
      if (pend >= 0) C.arena[pend] = make_int2((int)pend_ol, (int)r); // r is the older record
      else newest = (int)r;
      pend = (int)r;
      pend_ol = ax_ol;
      ++nrec;
    }
    if (cur < emit_end) {
      il = ax_il;
      base = prev_tok[ax_x & AUX_SRC];
      break;
    }
    cur = ax_x & AUX_SRC;
  }
  if (pend >= 0) C.arena[pend] = make_int2((int)pend_ol, base.bp);
  TokInfo t;
  t.hits = base.hits + hits;
  t.depth = base.depth + nrec;
  t.last_il = (int)il;
  t.bp = newest >= 0 ? newest : base.bp;
  return t;
}

// --- passes: one (cluster) barrier per pass -------------------------------
// What a pass leaves for the next one, read by every CTA after the pass's
// barrier (kills are written during the pass: kill words).
struct PassEnd {
  u32 row0_next; // rows so far: the next pass's first row
  u32 n_cand, n_app, eps_n;
  int error;
};

// After a pass's barrier: the counts of the pass (counter slot p = pass index
// mod 3, which every thread tracks); the slot of the pass after next (last
// read before this pass's barrier) is reset here.
template <int BLOCK, typename F, typename S>
__device__ PassEnd pass_end_c(const DecodeParams &P, const Chan<F, S> &C, Shared &sh, u32 p) {
  Counters &G = GC<F>(sh);
  if (threadIdx.x == 0) { // (the leader's counters: one thread per CTA loads them)
    sh.pe_row0 = G.flog_n;
    sh.pe_n_cand = G.n_cand[p];
    sh.pe_n_app = G.n_app[p];
    sh.pe_eps_n = G.eps_n;
    sh.pe_error = G.error;
    if (crank<F>() == 0) {
      const u32 z = p == 0 ? 2u : p - 1u; // (p + 2) mod 3
      G.n_cand[z] = 0;
      G.n_app[z] = 0;
    }
  }
  __syncthreads();
  PassEnd e;
  e.row0_next = sh.pe_row0;
  e.n_cand = sh.pe_n_cand;
  e.n_app = sh.pe_n_app;
  e.eps_n = sh.pe_eps_n;
  e.error = sh.pe_error;
  return e;
}

// _epsilon_rounds (decoder.py:250-316).  The frontier of the next round is
// the previous round's applications (n_front of them); the ones whose state
// has epsilon arcs are eps_list[lo, hi); row0 of each round is passed in
// (read after the previous pass's barrier).
template <int BLOCK, typename F, typename S>
__device__ void epsilon_rounds_c(const DecodeParams &P, const Chan<F, S> &C, Shared &sh, u32 lo, u32 hi,
                                 u32 n_front, u32 row0, u32 slot) {
  int rounds = 0;
  while (true) {
    if (!(n_front > 0 && rounds < P.max_eps)) {
      if (n_front > 0 && chan_t0<F>()) C.cs->info.eps_truncations += 1; // while-else 314-316
      break;
    }
    rounds++;
    if (chan_t0<F>()) GC<F>(sh).cnt_tok += n_front; // token expansions of the reference's round
    expand<BLOCK, exp_q<BLOCK>(), exp_u<F>(), false>(P, C, sh, C.eps_list + lo, hi - lo, row0, slot);
    PROF_MARK(sh, PF_EPS_X);
    PROF_COUNT(sh, PF_ROUNDS, 1);
    csync<F>();
    const PassEnd e = pass_end_c<BLOCK>(P, C, sh, slot);
    slot = slot == 2 ? 0u : slot + 1u;
    PROF_MARK(sh, PF_EPS_BAR);
    if (e.error) return;
    if (e.n_cand == 0 || e.n_app == 0) break; // decoder.py:263-265, 285-287
    lo = hi;
    hi = e.eps_n;
    n_front = e.n_app;
    row0 = e.row0_next;
  }
  // (no barrier: a pass ends with one, after which rows, kills, histograms
  // and minima are final, and the next reader, prune(), resets nothing)
}

// Provenance of a new token list (token i comes from frontier row rows[i]):
// resolve_row per token into the idle half of the provenance buffer (the
// previous list's provenance is still read through tok_info), then the halves
// swap.
template <int BLOCK, typename F, typename S>
__device__ void finish_tokens(const DecodeParams &P, const Chan<F, S> &C, Shared &sh, u32 n_tok,
                              const u32 *rows, int best_row) {
  // (max_depth, best_last_il and best_tok were reset by next_epoch())
  int md = 0;
  for (u32 i = crank<F>() * BLOCK + threadIdx.x; i < n_tok; i += BLOCK * F::cluster) {
    const u32 r = rows[i];
    const TokInfo t = resolve_row(P, C, sh, r, C.tok_info);
    md = max(md, t.depth);
    C.tok_info_alt[i] = t;
    if ((int)r == best_row) {
      GC<F>(sh).best_last_il = t.last_il;
      C.cs->best_tok = (int)i; // partial() reads it instead of another pass over the tokens
    }
  }
  md = __reduce_max_sync(0xFFFFFFFFu, md);
  if ((threadIdx.x & 31) == 0) atomicMax(&GC<F>(sh).max_depth, md);
  csync<F>();
  if (threadIdx.x == 0) {
    if (crank<F>() == 0) {
      C.cs->max_depth = GC<F>(sh).max_depth;
      C.cs->info.num_active = (int)n_tok;
      C.cs->tok_half ^= 1u;
    }
    Chan<F, S> &M = const_cast<Chan<F, S> &>(C); // every CTA's view swaps its halves
    TokInfo *t = M.tok_info;
    M.tok_info = M.tok_info_alt;
    M.tok_info_alt = t;
  }
  __syncthreads(); // the channel state above is read by peers after the caller's next cluster barrier
}

// Radix select over 64-bit keys (MSD, DB-bit digits, starting below the
// highest bit where the bounds [lo, hi] of all candidate keys differ).
// Returns t with count(key < t) < need <= count(key <= t).  On return
// `exact` tells whether ties at t still have to be resolved (then `need` is
// the number of keys equal to t that survive); otherwise every key <= t
// survives.  Each pass reads the keys QR per thread (loads first), into a
// 2^DB-bucket shared histogram.
template <int BLOCK, int QR, int DB, typename KeyFn>
__device__ u64 radix_select(Shared &sh, u32 *hist, u32 n, KeyFn keyf, u64 lo, u64 hi, u32 &need,
                            bool &exact) {
  const int tid = threadIdx.x;
  exact = true;
  if (lo == hi) return lo;
  int pos = 63 - __clzll(lo ^ hi);
  u64 prefix = pos >= 63 ? 0ull : (lo & ~((1ull << (pos + 1)) - 1));
  while (true) {
    const int lowbit = pos >= DB - 1 ? pos - (DB - 1) : 0;
    const int nb = pos - lowbit + 1;
    const u32 nbk = 1u << nb;
    const u64 above = pos >= 63 ? 0ull : ~((1ull << (pos + 1)) - 1);
    for (u32 b = tid; b < nbk; b += BLOCK) hist[b] = 0;
    __syncthreads();
    for (u32 base = 0; base < n; base += BLOCK * QR) {
      u64 kk[QR];
      bool ok[QR];
#pragma unroll
      for (int q = 0; q < QR; ++q) {
        const u32 i = base + q * BLOCK + tid;
        ok[q] = i < n;
        kk[q] = ok[q] ? keyf(i, ok[q]) : 0ull;
      }
#pragma unroll
      for (int q = 0; q < QR; ++q)
        if (ok[q] && (kk[q] & above) == prefix) atomicAdd(&hist[(kk[q] >> lowbit) & (nbk - 1)], 1u);
    }
    __syncthreads();
    // bucket holding the need-th key: contiguous bucket chunks per thread + block scan
    const u32 per = (nbk + BLOCK - 1) / BLOCK;
    const u32 b0 = min((u32)tid * per, nbk), b1 = min(b0 + per, nbk);
    u32 lsum = 0;
    for (u32 b = b0; b < b1; ++b) lsum += hist[b];
    u32 total;
    const u32 excl = block_excl_scan<BLOCK>(lsum, total, sh.scan);
    if (excl < need && need <= excl + lsum) {
      u32 cum = excl, b = b0;
      for (; b < b1; ++b) {
        if (cum + hist[b] >= need) break;
        cum += hist[b];
      }
      sh.sel = b;
      sh.cum = cum;
    }
    __syncthreads();
    const u32 b = sh.sel;
    need -= sh.cum;
    const u32 cnt = hist[b];
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
    PROF_COUNT(sh, PF_NPASS, 1);
  }
}

// _prune (decoder.py:319-334) + _best_token_pos (337-338) + silence
// bookkeeping (400-407) over the live rows of the frame's frontier log.  The
// frame's cost histogram (kept while rows were written and killed) gives the
// bucket holding the max_active-th live row within the beam; one pass over
// the rows (state, cost key) then takes every live row of a lower bucket
// (all within the beam) and sets the split bucket's rows within the beam
// aside (typically a few hundred), which are resolved exactly by (cost,
// state) with radix selects over their keys and then their states.  Bucket
// order is cost order, so the result is the exact top max_active.
template <int BLOCK, typename F, typename S>
__device__ bool prune(const DecodeParams &P, const Chan<F, S> &C, Shared &sh) {
  constexpr int QP = PRUNE_Q;
  constexpr u32 TILE = BLOCK * QP;
  // digit histograms of the split-bucket selection live in the expansion tile
  constexpr int DB = (BLOCK * exp_q<BLOCK>() >= 2048) ? 11 : (BLOCK * exp_q<BLOCK>() >= 1024) ? 10 : (BLOCK * exp_q<BLOCK>() >= 512) ? 9 : 8;
  const int tid = threadIdx.x;
  const u32 n_rows = GC<F>(sh).flog_n;
  const u64 best_ck = frame_min_ck<F>(C, sh);
  const double thr = key_cost(best_ck) + P.beam;
  const u64 thr_ck = cost_key(thr);
  u32 *scr_state = C.app_list; // (prune scratch)
  // split bucket: the first bucket where the live rows below and in it reach
  // max_active; buckets below the threshold's bucket are entirely in the beam
  const u32 bt = hbucket(sh, thr);
  const u32 want = (u32)P.max_active;
  // the frame's live-row histogram: this CTA's, or the sum over the cluster's
  const u32 *hist = sh.fhist;
  if constexpr (F::cluster > 1) {
    for (u32 b = tid; b < NB_HIST; b += BLOCK) {
      u32 t = 0;
#pragma unroll
      for (int r = 0; r < F::cluster; ++r) t += C.peer_sh[r]->fhist[b];
      C.t_a0[b] = t;
    }
    __syncthreads();
    hist = C.t_a0;
  }
  {
    constexpr u32 PER = NB_HIST / BLOCK > 0 ? NB_HIST / BLOCK : 1;
    const u32 b0 = min((u32)tid * PER, bt + 1), b1 = min(b0 + PER, bt + 1);
    u32 lsum = 0;
    for (u32 b = b0; b < b1; ++b) lsum += hist[b];
    u32 total;
    const u32 excl = block_excl_scan<BLOCK>(lsum, total, sh.scan);
    if (tid == 0) {
      sh.sel = bt;
      sh.cum = 0xFFFFFFFFu; // marks "not reached below bt"
    }
    __syncthreads();
    if (excl < want && want <= excl + lsum) {
      u32 cum = excl, b = b0;
      for (; b < b1; ++b) {
        if (cum + hist[b] >= want) break;
        cum += hist[b];
      }
      if (b < bt) {
        sh.sel = b;
        sh.cum = cum;
      }
    }
    __syncthreads();
  }
  const u32 split = sh.sel;
  u32 below = sh.cum; // live rows in buckets < split (when the split is below bt)
  // The frame's cutoff C* (the max_active-th cost, at most its bucket's upper
  // edge, or best + beam when the beam holds fewer rows): a filtered attempt
  // is exact iff C* <= its hint (advance()); otherwise the frame is redone.
  const double cut = split < bt ? fmin(thr, sh.hbase + ((double)split + 1.0001) / sh.hscale) : thr;
  const bool verified = !sh.filtered || cut <= sh.cut_hint;
  __syncthreads();
  if (!verified) {
    if (chan_t0<F>()) GC<F>(sh).cut_fail = cut;
    csync<F>();
    return false;
  }
  PROF_MARK(sh, PF_PHIST);
  if (tid == 0 && sh.next_row) { // the score row is read by the emitting pass only, which is now final
    bulk_row_load(const_cast<S *>(C.row), sh.next_row, (u32)(P.L * sizeof(S)), &sh.row_bar);
    sh.row_pending = 1;
  }
  if (tid == 0) { // every CTA keeps the cutoff history (its own copy; the channel state for later launches)
    Chan<F, S> &M = const_cast<Chan<F, S> &>(C);
    const double prev = M.prev_cut;
    const double rise = prev < INFINITY ? cut - prev : 0.0;
    M.cut_rise = fmax(rise, 0.8 * M.cut_rise);
    M.prev_cut = cut;
    M.prev_best = key_cost(best_ck);
    if (crank<F>() == 0) {
      C.cs->cut_rise = M.cut_rise;
      C.cs->prev_cut = cut;
      C.cs->prev_best = M.prev_best;
    }
  }
  // pass over the rows: survivors (bucket < split) -> token list; split
  // bucket within the beam -> set aside; best (cost, state)
  u64 bk = ~0ull;
  u32 bs = 0xFFFFFFFFu;
  int bi = -1;
  u32 n_tok = 0, n_mem = 0;
  u32 n_rec = 0; // the frame's emission records (rows with an output label, not displaced)
  u32 *mem_row = C.scr_row + P.flog_cap; // set-aside rows grow down from the top of scr_row
  for (u32 base = crank<F>() * TILE; base < n_rows; base += TILE * F::cluster) {
    // rows base + q * BLOCK + tid: warp-coalesced loads
    u32 st[QP], bq[QP];
    u64 ck[QP];
#pragma unroll
    for (int q = 0; q < QP; ++q) {
      const u32 i = base + (u32)q * BLOCK + (u32)tid;
      st[q] = i < n_rows ? C.flog_state[i] : ROW_DISP;
    }
#pragma unroll
    for (int q = 0; q < QP; ++q) {
      const u32 i = base + (u32)q * BLOCK + (u32)tid;
      ck[q] = i < n_rows ? C.flog_ck[i] : ~0ull;
    }
    {
#pragma unroll
      for (int q = 0; q < QP; ++q) {
        const u32 i = base + (u32)q * BLOCK + (u32)tid;
        const u32 kf = i < n_rows ? kill_flags(C, i) : ROW_DISP; // (beyond the rows: not live)
        n_rec += ((st[q] & ROW_REC) && !(kf & ROW_DISP)) ? 1u : 0u;
        st[q] = (st[q] & (ROW_STATE | ECODE_MASK)) | kf;
      }
    }
    u32 ns = 0, nm = 0;
#pragma unroll
    for (int q = 0; q < QP; ++q) {
      const bool live = !(st[q] & (ROW_DEAD | ROW_DISP));
      bq[q] = live ? hbucket(sh, key_cost(ck[q])) : NB_HIST;
      ns += (live && bq[q] < split) ? 1u : 0u;
      nm += (live && bq[q] == split && ck[q] <= thr_ck) ? 1u : 0u;
    }
    // both counts in one scan (survivors low, split-bucket rows high half:
    // a tile has at most BLOCK * QP of each, no carry between the halves)
    static_assert(BLOCK * QP < 65536, "packed prune scan");
    u32 tot_sm;
    const u32 psm = block_excl_scan<BLOCK>(ns | (nm << 16), tot_sm, sh.scan);
    const u32 tot_s = tot_sm & 0xFFFFu, tot_m = tot_sm >> 16;
    u32 ps = psm & 0xFFFFu;
    u32 pm = psm >> 16;
    if constexpr (F::cluster > 1) { // output positions reserved on the leader's counters
      if (tid == 0) {
        const unsigned long long b =
            tot_sm ? atomicAdd(&GC<F>(sh).out_tm, (unsigned long long)tot_s | ((unsigned long long)tot_m << 32)) : 0ull;
        sh.out_base_tok = (u32)b;
        sh.out_base_mem = (u32)(b >> 32);
      }
      __syncthreads();
      ps += sh.out_base_tok;
      pm += sh.out_base_mem;
      __syncthreads();
    } else {
      ps += n_tok;
      pm += n_mem;
    }
#pragma unroll
    for (int q = 0; q < QP; ++q) {
      if (bq[q] > split || (bq[q] == split && ck[q] > thr_ck)) continue;
      const u32 s = st[q] & ROW_STATE;
      const u32 sw = st[q] & (ROW_STATE | ECODE_MASK); // the token's state word keeps its ecode
      const u32 i = base + (u32)q * BLOCK + (u32)tid;
      if (ck[q] < bk || (ck[q] == bk && s < bs)) bk = ck[q], bs = s, bi = (int)i;
      if (bq[q] < split) {
        C.tok_state[ps] = sw;
        C.tok_cost[ps] = key_cost(ck[q]);
        C.scr_row[ps] = i;
        ++ps;
      } else {
        C.scr_key[pm] = ck[q];
        scr_state[pm] = sw;
        *(mem_row - 1 - pm) = i;
        ++pm;
      }
    }
    n_tok += tot_s;
    n_mem += tot_m;
  }
  PROF_MARK(sh, PF_PROWS);
  {
    n_rec = __reduce_add_sync(0xFFFFFFFFu, n_rec);
    if ((tid & 31) == 0 && n_rec) atomicAdd(&GC<F>(sh).n_rec_frame, (int)n_rec);
  }
  block_argmin<BLOCK>(bk, bs, bi, sh.redk, sh.reds, sh.redi);
  if constexpr (F::cluster == 1) { // (behind block_argmin's barriers)
    if (tid == 0 && sh.cnt.n_rec_frame) sh.cnt.rec_logical += (unsigned long long)sh.cnt.n_rec_frame;
  }
  if constexpr (F::cluster > 1) { // the cluster's best and totals
    // (peers read xbest_* and out_tok / out_mem, written again only in the
    // next attempt, behind more barriers: no second barrier here)
    if (tid == 0) {
      sh.xbest_k = bk;
      sh.xbest_s = bs;
      sh.xbest_i = bi;
    }
    csync<F>();
    for (int r = 0; r < F::cluster; ++r) {
      const Shared *o = C.peer_sh[r];
      const u64 k2 = o->xbest_k;
      const u32 s2 = o->xbest_s;
      if (k2 < bk || (k2 == bk && s2 < bs)) bk = k2, bs = s2, bi = o->xbest_i;
    }
    n_tok = GC<F>(sh).out_tok;
    n_mem = GC<F>(sh).out_mem;
    if (chan_t0<F>() && GC<F>(sh).n_rec_frame) // (rec_logical is the leader's own)
      GC<F>(sh).rec_logical += (unsigned long long)GC<F>(sh).n_rec_frame;
  }
  PROF_MARK(sh, PF_PRUNE_SCAN);
  if (below == 0xFFFFFFFFu) below = n_tok; // split at bt: everything below survives
  const u32 need = want > below ? want - below : 0u;
  if (n_mem > need) {
    if (n_tok + n_mem + need > P.flog_cap) { // survivors' rows would reach the set-aside rows
      if (chan_t0<F>()) set_error<F>(sh, E_CAP);
      csync<F>();
      return true;
    }
    // exact (cost, state) order inside the split bucket (a cluster's leader alone)
    if (crank<F>() == 0) {
    PROF_COUNT(sh, PF_NSEL, 1);
    PROF_COUNT(sh, PF_NMEM, n_mem);
    u64 tc = ~0ull;
    u32 ts = 0xFFFFFFFFu;
    // few rows (the usual case): each row's rank by (cost, state) among them,
    // compared 32 at a time through shuffles from a shared-memory copy
    const bool by_rank = n_mem <= RANK_MAX && n_mem <= BLOCK * (u32)exp_q<BLOCK>();
    u32 rank = 0xFFFFFFFFu;
    if (need > 0 && by_rank) {
      u64 *rk = reinterpret_cast<u64 *>(C.t_cost);
      u32 *rs = C.t_a0;
      u64 k = ~0ull;
      u32 s = 0xFFFFFFFFu;
      if ((u32)tid < n_mem) {
        k = C.scr_key[tid];
        s = scr_state[tid] & ROW_STATE;
        rk[tid] = k;
        rs[tid] = s;
      }
      __syncthreads();
      if (((u32)tid & ~31u) < n_mem) { // warps holding rows
        const u32 lane = (u32)tid & 31u;
        rank = 0;
        for (u32 c = 0; c < n_mem; c += 32) {
          const bool in = c + lane < n_mem;
          const u64 kc = in ? rk[c + lane] : ~0ull;
          const u32 sc = in ? rs[c + lane] : 0xFFFFFFFFu;
#pragma unroll 8
          for (int o = 0; o < 32; ++o) {
            const u64 ko = __shfl_sync(0xFFFFFFFFu, kc, o);
            const u32 so = __shfl_sync(0xFFFFFFFFu, sc, o);
            rank += (ko < k || (ko == k && so < s)) ? 1u : 0u;
          }
        }
      }
      PROF_COUNT(sh, PF_NPASS, 0);
    } else if (need > 0) {
      u32 nd = need;
      u64 lo = ~0ull, hi = 0ull;
      for (u32 m = tid; m < n_mem; m += BLOCK) {
        const u64 k = C.scr_key[m];
        lo = min(lo, k);
        hi = max(hi, k);
      }
      u32 dummy_s = 0;
      int dummy_i = 0;
      block_argmin<BLOCK>(lo, dummy_s, dummy_i, sh.redk, sh.reds, sh.redi);
      u64 nhi = ~hi;
      block_argmin<BLOCK>(nhi, dummy_s, dummy_i, sh.redk, sh.reds, sh.redi);
      hi = ~nhi;
      auto kf = [&](u32 i, bool &ok) -> u64 {
        ok = true;
        return C.scr_key[i];
      };
      bool exact;
      tc = radix_select<BLOCK, 8, DB>(sh, C.t_a0, n_mem, kf, lo, hi, nd, exact);
      if (exact) { // ties at the threshold cost: the smallest states survive
        auto sf = [&](u32 i, bool &ok) -> u64 {
          const u64 k = C.scr_key[i];
          const u32 s = scr_state[i] & ROW_STATE;
          ok = k == tc;
          return (u64)s;
        };
        bool exact2;
        ts = (u32)radix_select<BLOCK, 8, DB>(sh, C.t_a0, n_mem, sf, 0ull, 0xFFFFFFFFull, nd, exact2);
      }
    }
    for (u32 base = 0; base < n_mem; base += BLOCK) {
      const u32 m = base + tid;
      bool keep = false;
      u64 k = 0;
      u32 s = 0, r = 0;
      if (m < n_mem && need > 0) {
        k = C.scr_key[m];
        s = scr_state[m];
        r = *(mem_row - 1 - m);
        keep = by_rank ? rank < need : (k < tc || (k == tc && (s & ROW_STATE) <= ts));
      }
      u32 total;
      const u32 p = n_tok + block_excl_scan<BLOCK>(keep ? 1u : 0u, total, sh.scan);
      if (keep) {
        C.tok_state[p] = s;
        C.tok_cost[p] = key_cost(k);
        C.scr_row[p] = r;
      }
      n_tok += total;
    }
    if (F::cluster > 1 && tid == 0) GC<F>(sh).out_sel = n_tok;
    }
    csync<F>(); // the selected rows are tokens
    if constexpr (F::cluster > 1) n_tok = GC<F>(sh).out_sel;
  } else if (n_mem > 0) { // the whole split bucket survives (split across a cluster's CTAs)
    const u32 n0 = n_tok;
    for (u32 m = crank<F>() * BLOCK + tid; m < n_mem; m += BLOCK * F::cluster) {
      C.tok_state[n0 + m] = scr_state[m];
      C.tok_cost[n0 + m] = key_cost(C.scr_key[m]);
      C.scr_row[n0 + m] = *(mem_row - 1 - m);
    }
    n_tok += n_mem;
    csync<F>();
  }
  // (no split bucket: the row pass's tokens were published by its barrier)
  PROF_MARK(sh, PF_PRUNE_SEL);
  finish_tokens<BLOCK>(P, C, sh, n_tok, C.scr_row, bi);
  if (chan_t0<F>()) {
    if (P.silence_ilabel > 0 && GC<F>(sh).best_last_il == P.silence_ilabel)
      C.cs->info.trailing_silence += 1;
    else
      C.cs->info.trailing_silence = 0;
  }
  // (the channel state written above is read after advance()'s last barrier)
  PROF_MARK(sh, PF_PRUNE_OUT);
  return true;
}

// Token list := every live row of the epoch (after the utterance-start
// closure, which is not pruned).
template <int BLOCK, typename F, typename S>
__device__ void rows_to_tokens(const DecodeParams &P, const Chan<F, S> &C, Shared &sh) {
  const u32 n_rows = GC<F>(sh).flog_n;
  u32 n_tok = 0;
  csync<F>();
  // (a cluster's leader alone: the utterance start's closure is small)
  for (u32 i0 = 0; i0 < n_rows && crank<F>() == 0; i0 += BLOCK) {
    const u32 i = i0 + threadIdx.x;
    u32 st = i < n_rows ? C.flog_state[i] : ROW_DISP;
    const u32 kf = i < n_rows ? kill_flags(C, i) : ROW_DISP;
    const bool rec = (st & ROW_REC) && !(kf & ROW_DISP);
    st = (st & (ROW_STATE | ECODE_MASK)) | kf;
    const bool live = !(st & (ROW_DEAD | ROW_DISP));
    const u32 nrec = __popc(__ballot_sync(0xFFFFFFFFu, rec));
    if ((threadIdx.x & 31) == 0 && nrec) atomicAdd(&GC<F>(sh).rec_logical, (unsigned long long)nrec);
    u32 total;
    const u32 p = n_tok + block_excl_scan<BLOCK>(live ? 1u : 0u, total, sh.scan);
    if (live) {
      C.tok_state[p] = st & (ROW_STATE | ECODE_MASK);
      C.tok_cost[p] = key_cost(C.flog_ck[i]);
      C.scr_row[p] = i;
    }
    n_tok += total;
  }
  if constexpr (F::cluster > 1) {
    if (chan_t0<F>()) GC<F>(sh).out_tok = n_tok;
    csync<F>();
    n_tok = GC<F>(sh).out_tok;
  }
  csync<F>();
  finish_tokens<BLOCK>(P, C, sh, n_tok, C.scr_row, -1);
  if (threadIdx.x == 0) {
    Chan<F, S> &M = const_cast<Chan<F, S> &>(C);
    M.prev_best = key_cost(frame_min_ck<F>(C, sh));
    M.prev_cut = INFINITY; // the start closure is not pruned: no cutoff to start from
    M.cut_rise = 0.0;
    if (crank<F>() == 0) {
      C.cs->prev_best = M.prev_best;
      C.cs->prev_cut = INFINITY;
      C.cs->cut_rise = 0.0;
      C.cs->info.fresh = 0;
    }
  }
  csync<F>();
}

// Moves the channel to a fresh table epoch; the table is wiped when the
// 13-bit epoch tag would wrap, so a tag is never reused while stale values
// carrying it can still be in the table.  Also opens the frame's cost
// histogram: buckets of beam / HIST_PER_BEAM from one beam below the previous
// frame's best cost (values outside clamp into the end buckets).
//
// One cluster barrier: every CTA derives the epoch from its own view (C.epoch
// follows cs->epoch), and the counters reset here were last read by peers
// before an earlier cluster barrier (the previous frame's, or a redo's).
template <int BLOCK, typename F, typename S>
__device__ void next_epoch(const DecodeParams &P, Chan<F, S> &C, Shared &sh) {
  u32 e = C.epoch + 1;
  if ((e & 0x7FFFFFFFu) == 0) e = 0x100; // 31-bit key epochs (wrap also wipes below)
  if ((e & TAG_MASK) == 0) {
    if (F::hashed) {
      for (u32 i = threadIdx.x; i < P.table_cap; i += BLOCK) {
        C.table[i].key = 0;
        C.table[i].ck = 0;
        C.table[i].g = 0;
        C.table[i].info = 0;
      }
    } else {
      // (a cluster's CTAs each wipe their part: C.vals is this CTA's)
      uint4 *v = reinterpret_cast<uint4 *>(C.vals);
      const u32 part = (P.table_cap + F::cluster - 1) / F::cluster;
      for (u32 i = threadIdx.x; i < part; i += BLOCK) v[i] = make_uint4(0, 0, 0, 0);
      if (F::smem_table && C.gvals) { // keep the global table's tags consistent for later launches
        uint4 *gv = reinterpret_cast<uint4 *>(C.gvals);
        for (u32 i = crank<F>() * BLOCK + threadIdx.x; i < P.table_cap; i += BLOCK * F::cluster)
          gv[i] = make_uint4(0, 0, 0, 0);
      }
    }
    if (C.kill) // kill words carry the tag too
      for (u32 i = crank<F>() * BLOCK + threadIdx.x; i < P.flog_cap; i += BLOCK * F::cluster) C.kill[i] = 0;
    e += 1;
  }
  for (u32 b = threadIdx.x; b < NB_HIST; b += BLOCK) sh.fhist[b] = 0;
  __syncthreads(); // this CTA's threads have read C.epoch
  if (threadIdx.x == 0) {
    C.epoch = e;
    C.etag = e & TAG_MASK;
    sh.hbase = C.prev_best - P.beam;
    sh.hscale = HIST_PER_BEAM / P.beam;
    sh.cnt.min_ck = ~0ull; // every CTA's own frame minimum (frame_min_ck)
    sh.emit_end = 0;
  }
  if (chan_t0<F>()) {
    C.cs->epoch = e;
    GC<F>(sh).max_depth = 0; // finish_tokens()
    GC<F>(sh).best_last_il = 0;
    C.cs->best_tok = -1;
    GC<F>(sh).out_tm = 0;
    GC<F>(sh).n_new = 0;
    GC<F>(sh).n_app[0] = GC<F>(sh).n_app[1] = GC<F>(sh).n_app[2] = 0;
    GC<F>(sh).n_cand[0] = GC<F>(sh).n_cand[1] = GC<F>(sh).n_cand[2] = 0;
    GC<F>(sh).flog_n = 0;
    GC<F>(sh).eps_n = 0;
    GC<F>(sh).n_rec_frame = 0;
  }
  csync<F>();
}

// Copying collector for the emission arena: records reachable from the token
// list move to the other half, keeping their relative order, everything
// else (records of pruned or superseded tokens) is dropped.  Words never
// change: only record ids do, so the prefix-sharing path is reset.
template <int BLOCK, typename F, typename S>
__device__ void gc_arena(const DecodeParams &P, Chan<F, S> &C, Shared &sh) {
  const u32 n = GC<F>(sh).rec_n;
  const u32 nw = (n + 31) / 32;
  const u32 n_tok = (u32)C.cs->info.num_active;
  u32 carry = 0;
  csync<F>();
  if (crank<F>() == 0) { // a cluster's leader alone (rare)
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
  }
  csync<F>();
  if (threadIdx.x == 0) { // every CTA's view swaps the halves
    int2 *t = C.arena;
    C.arena = C.arena_to;
    C.arena_to = t;
    if (crank<F>() == 0) {
      GC<F>(sh).rec_n = carry;
      C.cs->arena_half ^= 1;
      C.cs->path_len = 0;
    }
  }
  csync<F>();
}

// Puts the utterance-start token into a fresh epoch (decoder.py:243-247):
// row 0, no source arc, always expanded by the closure.
template <int BLOCK, typename F, typename S>
__device__ void materialize_start(const DecodeParams &P, Chan<F, S> &C, Shared &sh) {
  next_epoch<BLOCK>(P, C, sh);
  if (chan_t0<F>()) {
    RelaxAcc acc;
    acc.min_ck = ~0ull;
    acc.n_new = acc.n_app = 0;
    acc.n_rec = 0;
    const bool on1[1] = {true};
    const u32 d1[1] = {(u32)P.start}, dc1[1] = {state_codes(P, (u32)P.start)}, g1[1] = {G_START}, s1[1] = {0u},
              f1[1] = {ROW_EPS}, z1[1] = {0u};
    const u64 c1[1] = {cost_key(0.0)};
    relax_batch<1>(P, C, sh, acc, on1, d1, dc1, c1, g1, s1, f1, z1, z1, 0u);
    GC<F>(sh).n_app[0] = GC<F>(sh).n_cand[0] = 0; // the closure's first round counts its own
    sh.cnt.min_ck = cost_key(0.0);
  }
  csync<F>();
}

// The leader's warp 0 writes the deferred partial hypothesis (the other
// warps go on; the caller's next cluster barrier publishes it).
template <typename F, typename S>
__device__ __forceinline__ void flush_pending(const DecodeParams &P, Chan<F, S> &C, Shared &sh, bool &pend) {
  if (pend && crank<F>() == 0 && threadIdx.x < 32) emit_pending_warp(P, C, sh);
  pend = false;
}

// advance_frame (decoder.py:341-411) for frame row C.row.  pend: a deferred
// partial hypothesis of the previous frame (cluster), written during this
// frame's emitting pass (or before the collector moves its records).
template <int BLOCK, typename F, typename S>
__device__ void advance(const DecodeParams &P, Chan<F, S> &C, Shared &sh, bool &pend) {
  ChanState *cs = C.cs;
  if (cs->info.status != AB_IDLE && cs->info.status != AB_DECODING) {
    if (chan_t0<F>()) set_error<F>(sh, E_STATUS);
    csync<F>();
    return;
  }
  // one frame appends at most flog_cap records: collect first if they might not fit
  if (!cs->info.fresh && (unsigned long long)GC<F>(sh).rec_n + P.flog_cap > P.arena_cap) {
    flush_pending(P, C, sh, pend); // (gc_arena begins with a cluster barrier)
    gc_arena<BLOCK>(P, C, sh);
    PROF_MARK(sh, PF_GC);
    if ((unsigned long long)GC<F>(sh).rec_n + P.flog_cap > P.arena_cap) {
      if (chan_t0<F>()) set_error<F>(sh, E_CAP);
      csync<F>();
      return;
    }
  }
  if (threadIdx.x == 0) C.ucut0 = C.ucut = INFINITY;
  // (no barrier: the channel state read below was written before the
  // previous frame's last cluster barrier; next_epoch() has the next one)
  if (cs->info.fresh) {
    flush_pending(P, C, sh, pend); // (none: a partial is deferred only while the utterance goes on)
    materialize_start<BLOCK>(P, C, sh);
    { // utterance-start closure (no prune): one row (the start token) so far
      const u32 hi0 = GC<F>(sh).eps_n;
      csync<F>();
      epsilon_rounds_c<BLOCK>(P, C, sh, 0u, hi0, 1u, 1u, 0u);
    }
    if (GC<F>(sh).error) return;
    rows_to_tokens<BLOCK>(P, C, sh); // (clears fresh; ends with a cluster barrier)
  }
  PROF_MARK(sh, PF_START);
  const u32 n_tok = (u32)cs->info.num_active;
  // Expansion-time cutoff.  No token whose cost exceeds the frame's cutoff C*
  // (min(best + beam, max_active-th cost)) survives prune, and an epsilon
  // path from a state lowers a cost by at most the context's slack S (-min
  // over states of the cheapest epsilon path from them: 0 without negative
  // epsilon weights).  So a candidate above U + S, for any U >= C*, is
  // neither a survivor nor on a survivor's path: dropping it leaves the
  // surviving tokens, their costs and their provenance exactly as the
  // reference computes them.  U is a hint (the previous frame's cutoff plus
  // its recent rise), verified after the closure: the filtered frame's own
  // cutoff C*_f >= C* (its candidates are a subset), so C*_f <= U proves the
  // frame exact; else the frame is redone (prune returns false before it has
  // written anything) with U = C*_f of the failed attempt, which keeps a
  // superset of its candidates and so verifies; a third attempt, should one
  // be needed, is unfiltered.  Emission records and epsilon-round
  // truncations of dropped candidates are not counted (P.exact keeps every
  // candidate and the reference's len(store) / eps_truncations).
  const unsigned long long c_tok = GC<F>(sh).cnt_tok, c_emit = GC<F>(sh).cnt_emit, c_eps = GC<F>(sh).cnt_eps;
  const long long eps_tr = cs->info.eps_truncations;
  bool filt = !P.exact && C.prev_cut < INFINITY && C.slack < INFINITY && P.beam < INFINITY &&
              P.max_eps <= C.slack_rounds;
  // (a peer may still read the status above: IDLE or DECODING, both pass)
  if (chan_t0<F>() && cs->info.status != AB_DECODING) cs->info.status = AB_DECODING;
  for (int attempt = 0;; ++attempt) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const double hint = !filt ? INFINITY
                          : attempt == 0 ? C.prev_cut + fmax(C.cut_rise, P.hint_min) + P.hint_extra +
                                               (cs->info.frame_index < P.hint_warm_frames ? P.hint_warm : 0.0)
                                         : GC<F>(sh).cut_fail;
      sh.cut_hint = hint;
      sh.filtered = filt ? 1 : 0;
      // (+ a margin for the f64 rounding of path sums)
      const double m = 1e-9 * fmax(1.0, fabs(hint));
      C.ucut0 = filt ? hint + m : INFINITY;
      C.ucut = filt ? hint + C.slack + m : INFINITY;
    }
    next_epoch<BLOCK>(P, C, sh);
    PROF_MARK(sh, PF_EPOCH);
    const bool skip0 = pend; // global warp 0 (the leader's warp 0) writes the pending hypothesis
    flush_pending(P, C, sh, pend);
    expand<BLOCK, exp_q<BLOCK>(), exp_u<F>(), true>(P, C, sh, nullptr, n_tok, 0u, 0u, skip0);
    PROF_MARK(sh, PF_EMIT_X);
    csync<F>();
    u32 n_app, eps_hi, row0_eps;
    int err;
    {
      const PassEnd e = pass_end_c<BLOCK>(P, C, sh, 0u);
      err = e.error;
      n_app = e.n_app;
      eps_hi = e.eps_n;
      row0_eps = e.row0_next;
      if (threadIdx.x == 0) sh.emit_end = e.row0_next; // read in resolve_row, behind more barriers
    }
    PROF_MARK(sh, PF_EMIT_BAR);
    if (err) return;
    bool ok = true;
    if (n_app == 0) {
      // no emitting arcs: every token dies (decoder.py:394-398); a filtered
      // attempt proves nothing here
      if (filt) ok = false;
      else if (chan_t0<F>()) cs->info.num_active = 0;
    } else {
      epsilon_rounds_c<BLOCK>(P, C, sh, 0u, eps_hi, n_app, row0_eps, 1u);
      PROF_MARK(sh, PF_EPS_S);
      if (GC<F>(sh).error) return;
      ok = prune<BLOCK>(P, C, sh);
    }
    if (ok) break;
    csync<F>();
    if (chan_t0<F>()) { // redo: undo the attempt's counters
      GC<F>(sh).cnt_tok = c_tok;
      GC<F>(sh).cnt_emit = c_emit;
      GC<F>(sh).cnt_eps = c_eps;
      cs->info.eps_truncations = eps_tr;
      cs->info.cut_redos += 1;
    }
    csync<F>();
    filt = filt && attempt == 0 && GC<F>(sh).cut_fail < INFINITY; // second attempt: hint = C*_f; third: none
  }
  if (threadIdx.x == 0) C.ucut0 = C.ucut = INFINITY;
  if (chan_t0<F>()) {
    cs->info.frame_index += 1;
    cs->info.total_frames += 1;
  }
  csync<F>();
  PROF_MARK(sh, PF_ADV_BAR);
}

// Traceback with prefix sharing against the channel's previous hypothesis
// path (EmissionStore.backtrace, decoder.py:95-102), by one thread: the new
// path's records and words from depth down to the first record the previous
// path has at the same depth; reserves the new words.  False: E_CAP (set).
template <typename F, typename S>
__device__ bool hyp_walk(const DecodeParams &P, Chan<F, S> &C, Shared &sh, int out_idx, int bp, int depth,
                         int &shared_words, long long &words_off) {
  ChanState *cs = C.cs;
  if ((u32)depth > P.path_cap) {
    set_error<F>(sh, E_CAP);
    return false;
  }
  int rec = bp, d = depth;
  const int plen = cs->path_len;
  PROF_COUNT(sh, PF_NHYP, 1);
  // (one dependent load per step: the record and the previous path's entry
  // at the same depth are loaded together)
  while (d > 0) {
    const int2 r = C.arena[rec];
    if (d <= plen && C.path_rec[d - 1] == rec) break;
    PROF_COUNT(sh, PF_WALK, 1);
    C.path_rec[d - 1] = rec;
    C.path_words[d - 1] = r.x;
    rec = r.y;
    --d;
  }
  shared_words = d;
  cs->path_len = depth;
  const long long need = depth - d;
  const long long off = P.words_used[C.b];
  if (off + need > P.words_stride || out_idx >= P.hyp_stride) {
    set_error<F>(sh, E_CAP);
    return false;
  }
  P.words_used[C.b] = off + need;
  words_off = (long long)C.b * P.words_stride + off;
  return true;
}

template <typename F, typename S>
__device__ __forceinline__ void write_hyp(const DecodeParams &P, const Chan<F, S> &C, int out_idx, int kind,
                                          int fallback, double cost, long long frame, int hits, int s0, int depth,
                                          long long off) {
  DevHyp h;
  h.cost = cost;
  h.frame = frame;
  h.kind = kind;
  h.fallback = fallback;
  h.hits = hits;
  h.shared = s0;
  h.n_words = depth;
  h.pad = 0;
  h.words_off = off;
  P.hyps[(size_t)C.b * P.hyp_stride + out_idx] = h;
}

// Hypothesis output by the whole CTA.
template <int BLOCK, typename F, typename S>
__device__ void emit_hyp(const DecodeParams &P, Chan<F, S> &C, Shared &sh, int out_idx, int kind, int fallback,
                         double cost, int bp, int depth, int hits) {
  if (threadIdx.x == 0) {
    int s0 = 0;
    long long off = 0;
    if (hyp_walk(P, C, sh, out_idx, bp, depth, s0, off)) {
      sh.shared_words = s0;
      sh.words_off = off;
    }
  }
  __syncthreads();
  if (GC<F>(sh).error) return;
  const int s0 = sh.shared_words;
  const long long off = sh.words_off;
  for (int i = s0 + threadIdx.x; i < depth; i += BLOCK) P.words[off + (i - s0)] = C.path_words[i];
  if (threadIdx.x == 0)
    write_hyp(P, C, out_idx, kind, fallback, cost, C.cs->info.total_frames, hits, s0, depth, off);
  __syncthreads();
}

// The best token (partial_hypothesis, decoder.py:414-423), by the whole CTA:
// false if the channel is dead (E_DEAD set).
template <int BLOCK, typename F, typename S>
__device__ bool partial_pick(const DecodeParams &P, Chan<F, S> &C, Shared &sh, PendHyp &h) {
  ChanState *cs = C.cs;
  h.frame = cs->info.total_frames;
  if (cs->info.fresh) {
    h.cost = 0.0;
    h.bp = -1;
    h.depth = 0;
    h.hits = 0;
    return true;
  }
  const u32 n = (u32)cs->info.num_active;
  if (n == 0) {
    if (threadIdx.x == 0) set_error<F>(sh, E_DEAD);
    __syncthreads();
    return false;
  }
  // the best (cost, state) token: prune found it (best_tok), else one pass
  int bi = cs->best_tok;
  if (bi < 0 || (u32)bi >= n) {
    u64 bk = ~0ull;
    u32 bs = 0xFFFFFFFFu;
    bi = -1;
    for (u32 i = threadIdx.x; i < n; i += BLOCK) {
      const u64 k = cost_key(C.tok_cost[i]);
      const u32 s = C.tok_state[i] & ROW_STATE;
      if (k < bk || (k == bk && s < bs)) bk = k, bs = s, bi = (int)i;
    }
    block_argmin<BLOCK>(bk, bs, bi, sh.redk, sh.reds, sh.redi);
  }
  const TokInfo t = C.tok_info[bi];
  h.cost = C.tok_cost[bi];
  h.bp = t.bp;
  h.depth = t.depth;
  h.hits = t.hits;
  return true;
}

// partial_hypothesis (decoder.py:414-423).
template <int BLOCK, typename F, typename S>
__device__ void partial(const DecodeParams &P, Chan<F, S> &C, Shared &sh, int out_idx) {
  PendHyp h;
  if (partial_pick<BLOCK>(P, C, sh, h)) emit_hyp<BLOCK>(P, C, sh, out_idx, AB_PARTIAL, 0, h.cost, h.bp, h.depth, h.hits);
}

// A cluster's deferred partial hypothesis (decode_kernel): picked at the end
// of its frame by the leader CTA, walked and written by the leader's warp 0
// while the rest of the cluster runs the next frame's emitting pass (its
// records and token provenance are not touched before that pass ends).
template <typename F, typename S>
__device__ void emit_pending_warp(const DecodeParams &P, Chan<F, S> &C, Shared &sh) {
  const PendHyp &h = sh.pend;
  const u32 lane = threadIdx.x & 31u;
  int s0 = 0, ok = 0;
  long long off = 0;
  if (lane == 0) ok = hyp_walk(P, C, sh, h.out_idx, h.bp, h.depth, s0, off) ? 1 : 0;
  __syncwarp();
  ok = __shfl_sync(0xFFFFFFFFu, ok, 0);
  if (!ok) return;
  s0 = __shfl_sync(0xFFFFFFFFu, s0, 0);
  off = __shfl_sync(0xFFFFFFFFu, off, 0);
  for (int i = s0 + (int)lane; i < h.depth; i += 32) P.words[off + (i - s0)] = C.path_words[i];
  if (lane == 0) write_hyp(P, C, h.out_idx, AB_PARTIAL, 0, h.cost, h.frame, h.hits, s0, h.depth, off);
  __syncwarp();
}

// finalize (decoder.py:426-460): best final token by (cost + final, state),
// falling back to the best token; then the utterance is reset.
template <int BLOCK, typename F, typename S>
__device__ void finalize(const DecodeParams &P, Chan<F, S> &C, Shared &sh, int out_idx) {
  ChanState *cs = C.cs;
  const int st = cs->info.status;
  if (st != AB_DECODING && st != AB_ENDPOINTED && !(st == AB_IDLE && cs->info.fresh)) {
    if (threadIdx.x == 0) set_error<F>(sh, E_STATUS);
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
      C.tok_state[0] = (u32)P.start | (ecode_of(state_codes(P, (u32)P.start)) << CODE_SHIFT);
      C.tok_cost[0] = 0.0;
      C.tok_info[0] = t;
      cs->info.num_active = 1;
      cs->info.fresh = 0;
    }
    __syncthreads();
  }
  const u32 n = (u32)cs->info.num_active;
  if (n == 0) {
    if (threadIdx.x == 0) set_error<F>(sh, E_DEAD);
    __syncthreads();
    return;
  }
  u64 fk = ~0ull, bk = ~0ull;
  u32 fs = 0xFFFFFFFFu, bs = 0xFFFFFFFFu;
  int fi = -1, bi = -1;
  for (u32 i = threadIdx.x; i < n; i += BLOCK) {
    const double c = C.tok_cost[i];
    const u32 s = C.tok_state[i] & ROW_STATE;
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
    cost = C.tok_cost[b] + __ldg(&P.final_cost[C.tok_state[b] & ROW_STATE]);
  } else {
    b = bi;
    fallback = 1;
    cost = C.tok_cost[b];
  }
  const TokInfo t = C.tok_info[b];
  emit_hyp<BLOCK>(P, C, sh, out_idx, AB_FINAL, fallback, cost, t.bp, t.depth, t.hits);
  if (GC<F>(sh).error) return;
  if (threadIdx.x == 0) {
    // _reset_utterance (decoder.py:151-159)
    cs->info.num_active = 0;
    cs->info.fresh = 1;
    cs->info.frame_index = 0;
    cs->info.trailing_silence = 0;
    GC<F>(sh).rec_n = 0;
    GC<F>(sh).rec_logical = 0;
    cs->path_len = 0;
    cs->max_depth = 0;
    cs->prev_cut = INFINITY;
    cs->info.utterance_index += 1;
    cs->info.status = AB_IDLE;
  }
  __syncthreads();
}

// The channel's view (pool pointers, context, epoch) lives in shared memory:
// it is uniform across the CTA, so keeping it out of registers frees them for
// in-flight loads.
template <int BLOCK, typename F, typename S>
__device__ void setup_channel(Chan<F, S> &C, const DecodeParams &P, int b, S *sh_row,
                              u32 *sh_ctx, u32 *t_a0 = nullptr, u32 *t_pref = nullptr,
                              double *t_cost = nullptr, u32 *t_src = nullptr, u32 *sh_neg = nullptr,
                              u32 *t_coarse = nullptr) {
  const int slot = P.slots[b];
  const int h = P.chans[slot].info.context;
  __syncthreads(); // the previous channel of this CTA is done with C
  if (threadIdx.x == 0) {
    C.P = &P;
    C.b = b;
    C.slot = slot;
    C.cs = &P.chans[slot];
    const size_t s = (size_t)slot;
    C.table = P.table ? P.table + s * P.table_cap : nullptr;
    C.vals = P.vals ? P.vals + 2 * s * P.table_cap : nullptr;
    C.gvals = C.vals;
    C.tok_state = P.tok_state + s * P.tok_cap;
    C.tok_cost = P.tok_cost + s * P.tok_cap;
    C.tok_info = P.tok_info + (2 * s + (C.cs->tok_half & 1u)) * P.tok_cap;
    C.tok_info_alt = P.tok_info + (2 * s + ((C.cs->tok_half & 1u) ^ 1u)) * P.tok_cap;
    C.flog_state = P.flog_state + s * P.flog_cap;
    C.flog_ck = P.flog_ck + s * P.flog_cap;
    C.flog_aux = P.flog_aux + s * P.flog_cap;
    C.eps_list = P.eps_list + s * P.flog_cap;
    C.app_list = P.app_list + s * P.flog_cap;
    C.kill = P.flog_kill ? P.flog_kill + s * P.flog_cap : nullptr;
    C.scr_key = P.scr_key + s * P.flog_cap;
    C.scr_row = P.scr_row + s * P.flog_cap;
    C.arena = P.arena + (2 * s + (C.cs->arena_half & 1)) * P.arena_cap;
    C.arena_to = P.arena + (2 * s + ((C.cs->arena_half & 1) ^ 1)) * P.arena_cap;
    C.gc_bits = P.gc_bits + s * (P.arena_cap / 32 + 1);
    C.gc_rank = P.gc_rank + s * (P.arena_cap / 32 + 1);
    C.path_rec = P.path_rec + s * P.path_cap;
    C.path_words = P.path_words + s * P.path_cap;
    C.row = sh_row;
    C.epoch = C.cs->epoch;
    C.prev_best = C.cs->prev_best;
    C.prev_cut = C.cs->prev_cut;
    C.cut_rise = C.cs->cut_rise;
    C.etag = C.epoch & TAG_MASK;
    C.ctx_mode = CTX_NONE;
    C.discount = 0.0;
    C.ctx_k = 0;
    C.ctx_lmask = 0;
    C.ctx_words = 0;
    C.ctx_list = nullptr;
    C.ctx_bits = nullptr;
    C.ctx_bits_x = nullptr;
    C.slack = P.slack0;
    C.slack_rounds = P.slack0_rounds;
    C.hq = nullptr;
    C.hq_unit = 0.0;
    C.fbits = C.fbits_x = nullptr;
    C.neg_fold = 0;
    C.ucut0 = C.ucut = INFINITY;
    C.neg = sh_neg;
    C.t_a0 = t_a0;
    C.t_pref = t_pref;
    C.t_cost = t_cost;
    C.t_src = t_src;
    C.t_coarse = t_coarse;
  }
  __syncthreads();
  if (h >= 0 && h < P.num_ctxs) {
    const CtxDesc d = P.ctxs[h];
    int mode = CTX_NONE;
    if (d.k == 0) {
      mode = CTX_NONE;
    } else if (d.mode == CTX_LABELS) {
      for (u32 i = threadIdx.x; i < d.words; i += BLOCK) sh_ctx[i] = d.bits[i];
      mode = CTX_LABELS;
    } else if (d.mode == CTX_BITSET) {
      mode = CTX_BITSET;
    } else if (d.mode == CTX_SLIST && d.words && d.words <= P.ctx_words_cap) {
      for (u32 i = threadIdx.x; i < d.words; i += BLOCK) sh_ctx[i] = d.hash[i]; // the Bloom filter
      mode = CTX_SLIST;
    } else {
      mode = CTX_GLIST;
    }
    if (threadIdx.x == 0) {
      C.discount = d.discount;
      C.ctx_k = d.k;
      C.ctx_lmask = d.lmask;
      C.ctx_mode = mode;
      C.ctx_words = d.words;
      C.ctx_bits = (mode == CTX_LABELS || mode == CTX_SLIST) ? sh_ctx : d.bits;
      C.ctx_bits_x = d.bits_x;
      if (mode != CTX_NONE) {
        C.slack = d.slack;
        C.slack_rounds = d.slack_rounds;
        C.hq = d.hq;
        C.hq_unit = d.hq_unit;
        C.fbits = d.fbits;
        C.fbits_x = d.fbits_x;
      }
      C.ctx_list = d.list;
    }
  }
  __syncthreads();
  if (C.slack > 0.0 && !C.hq) { // the neg Bloom filter of the weighting in use
    const u32 *src = P.neg0;
    if (h >= 0 && h < P.num_ctxs && P.ctxs[h].k) src = P.ctxs[h].neg;
    if (sh_neg && src) {
      const u32 W = P.neg_words;
      src += 2 * NEG_WORDS - 2 * W;
      for (u32 i = threadIdx.x; i < W; i += BLOCK) sh_neg[i] = src[i];
      if (threadIdx.x == 0) C.neg_fold = (u32)(__ffs(NEG_WORDS) - __ffs(W));
    } else if (threadIdx.x == 0) {
      C.slack = INFINITY; // no filter in this launch's layout: no cutoff for this channel
    }
  }
  __syncthreads();
}

// 64 registers per thread: 8 CTAs of 128 threads (or 4 x 256, 2 x 512) per SM.
// Persistent over channels: CTA i decodes batch entries i, i + grid, ... one
// after the other (the host sizes the grid so every CTA gets the same count).
template <int BLOCK, typename F, typename S>
#ifndef AB_MINB
#define AB_MINB 4
#endif
__global__ void __launch_bounds__(BLOCK, (AB_MINB * 256 / BLOCK) > 0 ? (AB_MINB * 256 / BLOCK) : 1)
    decode_kernel(const __grid_constant__ DecodeParams P) {
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  __shared__ Shared sh;
  __shared__ Chan<F, S> C;
  __shared__ double tile_cost[BLOCK * exp_q<BLOCK>()];
  __shared__ u32 tile_a0[BLOCK * exp_q<BLOCK>()];
  __shared__ u32 tile_pref[BLOCK * exp_q<BLOCK>() + 1];
  __shared__ u32 tile_src[BLOCK * exp_q<BLOCK>()];
  __shared__ u32 tile_coarse[BLOCK >= AB_WARP_TILES_MIN_BLOCK ? 1 : TILE_COARSE]; // CTA tiles only
  // dynamic: context words | score row | neg Bloom filter | (small graphs) the
  // channel's direct token table (host: launch_smem_layout, dyn_smem)
  u32 *sh_ctx = reinterpret_cast<u32 *>(dyn_smem);
  S *sh_row = reinterpret_cast<S *>(dyn_smem + P.ctx_words_cap * sizeof(u32));
  const bool row_in_smem = P.row_in_smem != 0;
  u32 *sh_neg = reinterpret_cast<u32 *>(dyn_smem + P.ctx_words_cap * sizeof(u32) +
                                        (row_in_smem ? ((size_t)P.L * sizeof(S) + 15) / 16 * 16 : 0));
  uint4 *sh_table = reinterpret_cast<uint4 *>(sh_neg + P.neg_words);
  if (threadIdx.x == 0) {
    mbar_init(&sh.row_bar);
    sh.row_phase = 0;
    sh.row_pending = 0;
    sh.next_row = nullptr;
  }
  // a channel per CTA, or per cluster of F::cluster CTAs (leader = rank 0)
  constexpr int CLU = F::cluster;
  const bool lead = crank<F>() == 0;
  const u32 part = (P.table_cap + CLU - 1) / CLU; // this CTA's share of a shared-memory table
  for (int b = blockIdx.x / CLU; b < P.n; b += gridDim.x / CLU) {
    setup_channel<BLOCK>(C, P, b, sh_row, sh_ctx, tile_a0, tile_pref, tile_cost, tile_src,
                         P.neg_words ? sh_neg : nullptr, tile_coarse);
    ChanState *cs = C.cs;
    if (F::smem_table) { // a fresh table per channel: zero tags are never current
      for (u32 i = threadIdx.x; i < part; i += BLOCK) sh_table[i] = make_uint4(0, 0, 0, 0);
    }
    if (threadIdx.x == 0) {
      if (F::smem_table) C.vals = reinterpret_cast<u64 *>(sh_table);
      if constexpr (CLU > 1) { // the leader's counters and every CTA's table part / Shared, over DSMEM
        namespace cg = cooperative_groups;
        cg::cluster_group cl = cg::this_cluster();
        sh.lead = cl.map_shared_rank(&sh.cnt, 0);
        for (int r = 0; r < CLU; ++r) {
          C.peer_vals[r] = reinterpret_cast<u64 *>(cl.map_shared_rank(sh_table, r));
          C.peer_sh[r] = cl.map_shared_rank(&sh, r);
        }
      }
    }
    if (chan_t0<F>()) {
      Counters &G = sh.cnt;
      G.error = 0;
      G.rec_n = cs->rec_phys;
      G.rec_logical = (unsigned long long)cs->info.store_len;
      G.cnt_tok = G.cnt_emit = G.cnt_eps = 0;
      G.n_new = G.flog_n = 0;
      G.n_app[0] = G.n_app[1] = G.n_app[2] = G.n_cand[0] = G.n_cand[1] = G.n_cand[2] = 0;
#ifdef AB_PROFILE
      for (int q = 0; q < PF_N; ++q) sh.prof[q] = 0;
      sh.prof_t = clock64();
#endif
    }
    csync<F>();
    const int T = P.frames[b];
    const S *scores = reinterpret_cast<const S *>(P.scores) + P.score_off[b];
    int n_out = 0;
    const bool was_finished = P.mode == AB_MODE_STREAM && cs->info.status == AB_FINISHED;
    csync<F>();
    if (was_finished && chan_t0<F>()) cs->info.status = AB_IDLE; // decoder.py:488-489
    csync<F>();
    int t = 0;
    bool pend = false; // a deferred partial hypothesis (cluster)
    for (; t < T; ++t) {
      if (P.mode == AB_MODE_STREAM) {
        // a frame adds at most 1 + max_eps words to any path (a fresh channel's
        // start closure up to max_eps more) and emits at most two hypotheses of
        // at most path_cap words; pause (the host relaunches) if they might not fit
        const long long E = min((long long)max(P.max_eps, 0), (long long)P.path_cap);
        const long long bound =
            min((long long)(cs->info.fresh ? E : cs->max_depth) + 2 + E, (long long)P.path_cap);
        if (P.words_used[b] + (pend ? 3 : 2) * bound > P.words_stride || n_out + 2 > P.hyp_stride) {
          if (t == 0 && chan_t0<F>()) set_error<F>(sh, E_CAP); // no progress possible
          break;
        }
      }
      const S *grow = scores + (size_t)t * P.L;
      if (row_in_smem) {
        if (sh.row_pending) { // bulk-copied during the previous frame
          mbar_wait(&sh.row_bar, sh.row_phase);
        } else {
          for (int i = threadIdx.x; i < P.L; i += BLOCK) sh_row[i] = grow[i];
        }
      } else if (threadIdx.x == 0) {
        C.row = grow;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        if (sh.row_pending) {
          sh.row_pending = 0;
          sh.row_phase ^= 1u;
        }
        // the next row goes by bulk copy when it is 16-byte sized and aligned
        const S *nrow = grow + P.L;
        sh.next_row = (row_in_smem && t + 1 < T && ((P.L * sizeof(S)) & 15) == 0 &&
                       (reinterpret_cast<size_t>(nrow) & 15) == 0) ? nrow : nullptr;
      }
      __syncthreads(); // (the row and next_row are this CTA's)
      PROF_MARK(sh, PF_ROW);
      advance<BLOCK>(P, C, sh, pend);
      if (GC<F>(sh).error) break;
      if (P.mode == AB_MODE_STREAM) {
        // hypotheses: the leader CTA alone (every CTA counts them)
        if (cs->info.frame_index % P.partial_every == 0) {
          // a cluster defers the traceback to the next frame's emitting pass
          // while the utterance goes on (every CTA decides alike)
          const bool defer = F::cluster > 1 && t + 1 < T && cs->info.trailing_silence < P.endpoint_silence_frames &&
                             (cs->info.fresh || cs->info.num_active > 0);
          if (defer) {
            if (lead) {
              PendHyp h;
              partial_pick<BLOCK>(P, C, sh, h);
              if (threadIdx.x == 0) {
                h.out_idx = n_out;
                sh.pend = h; // (read by this CTA's warp 0, behind a CTA barrier)
              }
            }
            pend = true;
            ++n_out;
          } else {
            if (lead) partial<BLOCK>(P, C, sh, n_out);
            ++n_out;
            csync<F>();
            if (GC<F>(sh).error) break;
          }
        }
        if (cs->info.trailing_silence >= P.endpoint_silence_frames) { // detect_endpoint 463-464
          if (chan_t0<F>()) cs->info.status = AB_ENDPOINTED;
          __syncthreads(); // (finalize() runs in the leader CTA, which wrote the status)
          if (lead) finalize<BLOCK>(P, C, sh, n_out);
          ++n_out;
          csync<F>();
          if (GC<F>(sh).error) break;
        }
      }
      // (no barrier: advance() and each hypothesis end with one)
      PROF_MARK(sh, PF_HYP);
    }
    if (pend) { // the last deferred hypothesis
      flush_pending(P, C, sh, pend);
      csync<F>();
    }
    if (sh.row_pending) { // a prefetched row nobody will read: let it land before the buffer is reused
      mbar_wait(&sh.row_bar, sh.row_phase);
      __syncthreads();
      if (threadIdx.x == 0) {
        sh.row_pending = 0;
        sh.row_phase ^= 1u;
      }
    }
    csync<F>();
    const bool done = t == T;
    if (P.mode == AB_MODE_STREAM && !GC<F>(sh).error && done && P.final_chunk) {
      // decoder.py:498-501: final hypothesis if frames were consumed or the stream is empty
      const bool fin = cs->info.frame_index > 0 || P.stream_frames[b] == 0;
      csync<F>();
      if (fin) {
        if (lead) finalize<BLOCK>(P, C, sh, n_out);
        ++n_out;
      }
      csync<F>();
      if (!GC<F>(sh).error && chan_t0<F>()) cs->info.status = AB_FINISHED;
    }
    csync<F>();
    if (chan_t0<F>()) {
      cs->rec_phys = GC<F>(sh).rec_n;
      cs->info.store_len = (long long)GC<F>(sh).rec_logical;
      cs->info.tok_expansions += GC<F>(sh).cnt_tok;
      cs->info.emit_arcs += GC<F>(sh).cnt_emit;
      cs->info.eps_arcs += GC<F>(sh).cnt_eps;
      cs->info.error = GC<F>(sh).error;
      P.n_hyps[b] = n_out;
      P.errors[b] = GC<F>(sh).error;
      P.frames_done[b] = t;
#ifdef AB_PROFILE
      for (int q = 0; q < PF_N; ++q) atomicAdd(&P.prof[q], sh.prof[q]);
#endif
    }
    csync<F>(); // no CTA of the cluster reuses its shared memory while a peer may still read it
  }
}

// Standalone partial / finalize for one channel (the per-call Python API).
template <int BLOCK, typename F, typename S>
__global__ void __launch_bounds__(BLOCK) hyp_kernel(const __grid_constant__ DecodeParams P, int which) {
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  __shared__ Shared sh;
  u32 *sh_ctx = reinterpret_cast<u32 *>(dyn_smem);
  S *sh_row = reinterpret_cast<S *>(dyn_smem + CTX_SMEM_WORDS * sizeof(u32));
  __shared__ Chan<F, S> C;
  setup_channel<BLOCK>(C, P, (int)blockIdx.x, sh_row, sh_ctx);
  if (threadIdx.x == 0) {
    GC<F>(sh).error = 0;
    GC<F>(sh).rec_n = C.cs->rec_phys;
    GC<F>(sh).rec_logical = (unsigned long long)C.cs->info.store_len;
  }
  __syncthreads();
  if (which == AB_PARTIAL) partial<BLOCK>(P, C, sh, 0);
  else finalize<BLOCK>(P, C, sh, 0);
  __syncthreads();
  if (threadIdx.x == 0) {
    C.cs->rec_phys = GC<F>(sh).rec_n;
    C.cs->info.store_len = (long long)GC<F>(sh).rec_logical;
    P.n_hyps[C.b] = GC<F>(sh).error ? 0 : 1;
    P.errors[C.b] = GC<F>(sh).error;
  }
}

} // namespace ab
