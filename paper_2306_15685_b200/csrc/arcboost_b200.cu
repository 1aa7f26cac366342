// arcboost-b200: C ABI (include/arcboost_b200.h) over the sm_100a decode kernels.
//
// Host responsibilities: build the device graph (split emitting / epsilon CSR,
// fst.py:165-191), the context store (biasing.py:86-117), per-channel device
// pools, launch the batch kernel, relaunch channels that paused for output
// space, pack hypotheses and words into one contiguous D2H transfer.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <sys/stat.h>

#include "context_compiler.h"
#include "graph_ingest.h"
#include "score_ingest.h"
#include "scoring.h"
#include "score_gen.cuh"
#include "decode_kernel.cuh"
#include "decode_instances.h"

// compiled in csrc/kernels/*.cu
AB_DECODE_ALL(AB_DECODE_EXTERN)

using namespace ab;

static thread_local std::string g_err;

static int fail(int code, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) return fail(AB_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

template <typename T> static cudaError_t dmalloc(T **p, size_t count, size_t &acc) {
  size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
  acc += bytes;
  return cudaMalloc((void **)p, bytes);
}

struct HostCtx {
  bool live = false;
  double discount = 0.0;
  u32 k = 0;
  int mode = CTX_SLIST; // device CTX_* code
  int abi_mode = AB_CTX_LIST;
  u32 words = 0;
  u32 *d_list = nullptr;   // the arc ids as an open-addressing set (list_slot; ~0 = empty)
  u32 list_mask = 0;       // its size - 1
  u32 *d_hash = nullptr; // CTX_SLIST: Bloom filter of the ids (words words)
  u32 *d_bits = nullptr;   // CTX_BITSET: emitting record positions; CTX_LABELS: olabel bitmap
  u32 *d_bits_x = nullptr; // CTX_BITSET: epsilon record positions
  double slack = 0.0;      // eps_slack of the context's weighting
  int slack_rounds = 0;
  u32 *d_neg = nullptr;    // its neg Bloom filters (NEG_BLOCK_WORDS)
  u32 neg_count = 0;       // states they flag
  u32 *d_hq = nullptr;     // or 2-bit per-state slack (dense contexts)
  u32 *d_fbits = nullptr, *d_fbits_x = nullptr; // dense contexts: per record position, "hq of the destination > 0"
  double hq_unit = 0.0;
};

struct ab_graph {
  int device = 0;
  int start = 0;
  int num_states = 0;
  int64_t num_arcs = 0;
  int L = 0;
  bool w32 = true;
  bool fmt16 = true; // f32 weights and 16-bit labels: 16-byte arc records
  std::vector<int32_t> olabels; // host copy for context classification
  std::vector<u32> ol_count;    // arcs per output label (empty if labels are huge)
  // device record position of every arc (bit 31 = epsilon array): BITSET
  // contexts are stored by record position, so the kernel's boost lookup is
  // addressed before the arc record arrives (issued next to the record load)
  std::vector<u32> arc_pos;
  std::vector<u32> arc_dst;      // next state of every arc (dense contexts' slack flags by position)
  uint64_t e_tot = 0, x_tot = 0; // records in the emitting / epsilon arrays
  // epsilon subgraph on the host (arc ids increasing; reverse adjacency by
  // destination) for the epsilon slack of a weighting (eps_slack)
  std::vector<u32> xe_g, xe_src, xe_dst, xr_off, xr_arc;
  std::vector<u32> xe_neg; // epsilon arcs with a negative graph weight
  std::vector<double> xe_w;
  std::vector<double> h_buf; // eps_slack scratch, one value per state
  double slack0 = 0.0;       // slack of the unbiased graph
  int slack0_rounds = 0;
  u32 *d_neg0 = nullptr;     // its neg Bloom filters (NEG_BLOCK_WORDS)
  u32 neg0_count = 0;        // states they flag
  uint2 *e_rng = nullptr, *x_rng = nullptr; // per state {begin, end}: one 8-byte request
  unsigned char *deg = nullptr;              // per state arc counts (DecodeParams::deg)
  void *e_arcs = nullptr, *x_arcs = nullptr;
  double *final_cost = nullptr;
  size_t bytes = 0;
  std::vector<HostCtx> ctxs;
  CtxDesc *d_ctxs = nullptr;
  size_t d_ctxs_cap = 0;
  cudaStream_t stream = nullptr;
};

struct ab_decoder {
  ab_graph *g = nullptr;
  int device = 0;
  int max_ch = 0;
  std::vector<int32_t> slot_ctx; // context handle of every slot (host mirror: sizes shared memory)
  ab_capacity cap{};
  u32 table_cap = 0;
  int hashed = 0;
  u32 tok_cap = 0, flog_cap = 0, arena_cap = 0, path_cap = 0;
  size_t bytes = 0;
  ChanState *chans = nullptr;
  Entry *table = nullptr;  // hashed
  u64 *vals = nullptr;     // direct
  u32 *tok_state = nullptr;
  double *tok_cost = nullptr;
  TokInfo *tok_info = nullptr;
  u32 *flog_state = nullptr;
  u64 *flog_ck = nullptr;
  uint4 *flog_aux = nullptr;
  uint4 *eps_list = nullptr;
  u32 *app_list = nullptr;
  u32 *flog_kill = nullptr; // kill words (decode_kernel.cuh KW_*)
  u64 *scr_key = nullptr;
  u32 *scr_row = nullptr;
  int2 *arena = nullptr;
  u32 *gc_bits = nullptr, *gc_rank = nullptr;
  int *path_rec = nullptr, *path_words = nullptr;
  // per-call buffers (grown on demand)
  size_t batch_cap = 0;
  int *d_slots = nullptr, *d_frames = nullptr, *d_sframes = nullptr, *d_nhyps = nullptr, *d_errors = nullptr,
      *d_done = nullptr;
  long long *d_soff = nullptr, *d_wused = nullptr;
  size_t hyps_cap = 0;
  DevHyp *d_hyps = nullptr;
  size_t words_cap = 0;
  int *d_words = nullptr;
  size_t packh_cap = 0, packw_cap = 0;
  DevHyp *d_packh = nullptr;
  int *d_packw = nullptr;
  long long *d_packoff = nullptr; // [2n]
  size_t stage_cap = 0;
  void *d_stage = nullptr; // two chunk buffers of host score rows (end-to-end path)
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copy[2] = {nullptr, nullptr};
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  float last_ms = 0.f;
  int last_launches = 0;
  size_t info_cap = 0;
  ab_channel_info *d_infos = nullptr;
  int *d_islots = nullptr;
  // accumulated results of the last ab_decode
  std::vector<int> res_nhyps, res_err;
  std::vector<std::vector<ab_hyp>> res_hyps;
  std::vector<std::vector<int32_t>> res_words;
};

extern "C" const char *ab_last_error(void) { return g_err.c_str(); }

extern "C" int ab_device_count(int32_t *count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    return fail(AB_ERR_CUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  *count = n;
  return AB_OK;
}

// ------------------------------------------------------------------ graph

static double eps_slack(ab_graph *g, const std::vector<u32> &boosted, double discount,
                        std::vector<u32> *neg_bits, int *rounds_ok, std::vector<u32> *hq = nullptr,
                        double *hq_unit = nullptr, u32 *neg_count = nullptr);

extern "C" int ab_graph_create(int32_t device, int32_t start, int32_t num_states,
                               int64_t num_arcs, const int64_t *row_offsets,
                               const int32_t *ilabels, const int32_t *olabels,
                               const int32_t *next_states, const double *weights,
                               int32_t num_finals, const int32_t *final_states,
                               const double *final_costs, ab_graph **out) {
  *out = nullptr;
  if (num_states < 1) return fail(AB_ERR_INVALID, "graph must have at least one state");
  if (num_arcs < 0 || num_arcs >= (int64_t)G_MASK) // arc ids carry a flag in bit 31
    return fail(AB_ERR_INVALID, "num_arcs %lld out of range", (long long)num_arcs);
  if (num_states > (int32_t)ROW_STATE)
    return fail(AB_ERR_INVALID, "too many states (max %u)", ROW_STATE);
  if (start < 0 || start >= num_states)
    return fail(AB_ERR_INVALID, "start state %d out of range for %d states", start, num_states);
  if (row_offsets[0] != 0 || row_offsets[num_states] != num_arcs)
    return fail(AB_ERR_INVALID, "row_offsets must start at 0 and end at num_arcs");
  for (int s = 0; s < num_states; ++s)
    if (row_offsets[s + 1] < row_offsets[s])
      return fail(AB_ERR_INVALID, "row_offsets not monotone at state %d", s);
  int L = 0;
  int max_ol = 0;
  bool w32 = true;
  std::vector<u32> e_cnt(num_states + 1, 0), x_cnt(num_states + 1, 0);
  for (int s = 0; s < num_states; ++s) {
    for (int64_t a = row_offsets[s]; a < row_offsets[s + 1]; ++a) {
      if (ilabels[a] < 0 || olabels[a] < 0)
        return fail(AB_ERR_INVALID, "negative label on arc %lld", (long long)a);
      if (next_states[a] < 0 || next_states[a] >= num_states)
        return fail(AB_ERR_INVALID, "arc %lld to nonexistent state %d", (long long)a,
                    next_states[a]);
      if (!std::isfinite(weights[a]))
        return fail(AB_ERR_INVALID, "non-finite weight on arc %lld", (long long)a);
      if ((double)(float)weights[a] != weights[a]) w32 = false;
      L = std::max(L, ilabels[a]);
      max_ol = std::max(max_ol, olabels[a]);
      if (ilabels[a] != 0) e_cnt[s + 1]++;
      else x_cnt[s + 1]++;
    }
  }
  for (int s = 0; s < num_states; ++s) {
    e_cnt[s + 1] += e_cnt[s];
    x_cnt[s + 1] += x_cnt[s];
  }
  std::vector<double> fin(num_states, std::nan(""));
  for (int i = 0; i < num_finals; ++i) {
    int s = final_states[i];
    if (s < 0 || s >= num_states) return fail(AB_ERR_INVALID, "final state %d out of range", s);
    if (!std::isfinite(final_costs[i]))
      return fail(AB_ERR_INVALID, "non-finite final weight at state %d", s);
    fin[s] = final_costs[i];
  }
  ab_graph *g = new ab_graph();
  g->device = device;
  g->start = start;
  g->num_states = num_states;
  g->num_arcs = num_arcs;
  g->L = L;
  g->w32 = w32;
  g->fmt16 = w32 && L <= 0xFFFF && max_ol <= 0xFFFF;
  g->olabels.assign(olabels, olabels + num_arcs);
  if (max_ol < (1 << 24)) {
    g->ol_count.assign((size_t)max_ol + 1, 0);
    for (int64_t a = 0; a < num_arcs; ++a) g->ol_count[olabels[a]]++;
  }
  cudaError_t ce = cudaSetDevice(device);
  if (ce != cudaSuccess) {
    delete g;
    return fail(AB_ERR_CUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(ce));
  }
  // build the split arc arrays (arc order inside each state preserved).
  // A state with at most SLOT_E emitting (SLOT_X epsilon) arcs keeps them in
  // its fixed slot at s * SLOT_E (s * SLOT_X), so the kernel finds them from
  // the state id and a 1-byte count that stays in L2, without a dependent
  // read of the range array; bigger states go to an overflow area after the
  // slots and are found through the ranges.  (Slots are skipped when they
  // would cost more than 8 GB.)  Overflow blocks, Fmt16: a block of up to
  // four 16-B records never straddles a 64-byte DRAM atom, longer blocks
  // start on an atom.
  const bool f16 = g->fmt16;
  size_t esz = f16 ? sizeof(EArc16) : sizeof(EArc24);
  size_t xsz = f16 ? sizeof(XArc16) : sizeof(XArc24);
  const bool slots = (uint64_t)num_states * (SLOT_E * esz + SLOT_X * xsz) <= (8ull << 30);
  std::vector<u32> e_beg(num_states), x_beg(num_states);
  std::vector<unsigned char> deg(num_states);
  uint64_t e_tot = slots ? (uint64_t)num_states * SLOT_E : 0, x_tot = slots ? (uint64_t)num_states * SLOT_X : 0;
  auto place = [&](uint64_t &cur, u32 cnt) -> u32 {
    if (f16 && cnt) {
      constexpr uint64_t ATOM = 4; // records per 64-byte atom
      if (cnt > ATOM || (cur % ATOM) + cnt > ATOM) cur = (cur + ATOM - 1) / ATOM * ATOM;
    }
    const u32 b = (u32)cur;
    cur += cnt;
    return b;
  };
  for (int s = 0; s < num_states; ++s) {
    const u32 ec = e_cnt[s + 1] - e_cnt[s], xc = x_cnt[s + 1] - x_cnt[s];
    u32 de = DEG_OVF, dx = DEG_OVF;
    if (slots && ec <= SLOT_E) {
      e_beg[s] = (u32)s * SLOT_E;
      de = ec;
    } else {
      e_beg[s] = place(e_tot, ec);
    }
    if (slots && xc <= SLOT_X) {
      x_beg[s] = (u32)s * SLOT_X;
      dx = xc;
    } else {
      x_beg[s] = place(x_tot, xc);
    }
    deg[s] = (unsigned char)(de | (dx << 4));
  }
  if (e_tot >= 0xFFFFFFFFull || x_tot >= 0xFFFFFFFFull) {
    delete g;
    return fail(AB_ERR_INVALID, "too many arcs after block alignment");
  }
  std::vector<unsigned char> eh(std::max<size_t>(e_tot, 1) * esz, 0), xh(std::max<size_t>(x_tot, 1) * xsz, 0);
  g->e_tot = e_tot;
  g->x_tot = x_tot;
  g->arc_pos.resize(num_arcs);
  g->arc_dst.resize(num_arcs);
  // a record's next-state word carries the destination's degree codes
  // (decode_kernel.cuh CODE_SHIFT): the kernel never loads the degree array
  auto codes = [&](int t) -> u32 {
    const u32 e = (u32)(deg[t] & 15u), x = (u32)(deg[t] >> 4);
    return ((e == DEG_OVF ? ECODE_OVF : e) | ((x == DEG_OVF ? XCODE_OVF : x) << 3)) << CODE_SHIFT;
  };
  for (int s = 0; s < num_states; ++s) {
    u32 pe = e_beg[s], px = x_beg[s];
    for (int64_t a = row_offsets[s]; a < row_offsets[s + 1]; ++a) {
      const int dst = next_states[a];
      g->arc_dst[a] = (u32)dst;
      const bool dst_eps = x_cnt[dst + 1] > x_cnt[dst];
      const u32 nsw = (u32)dst | codes(dst);
      if (ilabels[a] != 0) {
        const u32 ga = (u32)a | (dst_eps ? G_DEST_EPS : 0u);
        if (f16) {
          EArc16 r{nsw, ga, (float)weights[a],
                   (u32)ilabels[a] | ((u32)olabels[a] << 16)};
          memcpy(&eh[(size_t)pe * esz], &r, esz);
        } else {
          EArc24 r{nsw, ga, (u32)ilabels[a], (u32)olabels[a], weights[a]};
          memcpy(&eh[(size_t)pe * esz], &r, esz);
        }
        g->arc_pos[a] = pe;
        pe++;
      } else {
        const u32 ga = (u32)a | (dst_eps ? G_DEST_EPS : 0u);
        if (f16) {
          XArc16 r{nsw, ga, (float)weights[a], (u32)olabels[a]};
          memcpy(&xh[(size_t)px * xsz], &r, xsz);
        } else {
          XArc24 r{nsw, ga, (u32)olabels[a], 0u, weights[a]};
          memcpy(&xh[(size_t)px * xsz], &r, xsz);
        }
        g->arc_pos[a] = px | 0x80000000u;
        px++;
      }
    }
  }
  for (int s = 0; s < num_states; ++s)
    for (int64_t a = row_offsets[s]; a < row_offsets[s + 1]; ++a)
      if (ilabels[a] == 0) {
        g->xe_g.push_back((u32)a);
        g->xe_src.push_back((u32)s);
        g->xe_dst.push_back((u32)next_states[a]);
        if (weights[a] < 0.0) g->xe_neg.push_back((u32)g->xe_w.size());
        g->xe_w.push_back(weights[a]);
      }
  g->xr_off.assign((size_t)num_states + 1, 0);
  for (u32 d : g->xe_dst) g->xr_off[d + 1]++;
  for (int s = 0; s < num_states; ++s) g->xr_off[s + 1] += g->xr_off[s];
  g->xr_arc.resize(g->xe_g.size());
  {
    std::vector<u32> fill(g->xr_off.begin(), g->xr_off.end() - 1);
    for (size_t i = 0; i < g->xe_g.size(); ++i) g->xr_arc[fill[g->xe_dst[i]]++] = (u32)i;
  }
  std::vector<u32> neg0;
  g->slack0 = eps_slack(g, {}, 0.0, &neg0, &g->slack0_rounds, nullptr, nullptr, &g->neg0_count);
  size_t acc = 0;
  unsigned char *de = nullptr, *dx = nullptr;
  std::vector<uint2> erng(num_states), xrng(num_states);
  for (int s = 0; s < num_states; ++s) {
    erng[s] = make_uint2(e_beg[s], e_beg[s] + (e_cnt[s + 1] - e_cnt[s]));
    xrng[s] = make_uint2(x_beg[s], x_beg[s] + (x_cnt[s + 1] - x_cnt[s]));
  }
  if (dmalloc(&g->e_rng, num_states, acc) || dmalloc(&g->x_rng, num_states, acc) ||
      dmalloc(&de, eh.size(), acc) || dmalloc(&dx, xh.size(), acc) ||
      dmalloc(&g->final_cost, num_states, acc) || dmalloc(&g->deg, num_states, acc)) {
    ab_graph_destroy(g);
    return fail(AB_ERR_CUDA, "device allocation for the graph failed (%zu bytes)", acc);
  }
  g->e_arcs = de;
  g->x_arcs = dx;
  if (dmalloc(&g->d_neg0, NEG_BLOCK_WORDS, acc) ||
      cudaMemcpy(g->d_neg0, neg0.data(), NEG_BLOCK_WORDS * sizeof(u32), cudaMemcpyHostToDevice) != cudaSuccess) {
    ab_graph_destroy(g);
    return fail(AB_ERR_CUDA, "device allocation for the graph failed");
  }
  g->bytes = acc;
  if (cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMemcpy(g->e_rng, erng.data(), num_states * sizeof(uint2), cudaMemcpyHostToDevice) ||
      cudaMemcpy(g->x_rng, xrng.data(), num_states * sizeof(uint2), cudaMemcpyHostToDevice) ||
      cudaMemcpy(de, eh.data(), eh.size(), cudaMemcpyHostToDevice) ||
      cudaMemcpy(dx, xh.data(), xh.size(), cudaMemcpyHostToDevice) ||
      cudaMemcpy(g->final_cost, fin.data(), num_states * sizeof(double), cudaMemcpyHostToDevice) ||
      cudaMemcpy(g->deg, deg.data(), num_states, cudaMemcpyHostToDevice)) {
    ab_graph_destroy(g);
    return fail(AB_ERR_CUDA, "graph upload failed: %s", cudaGetErrorString(cudaGetLastError()));
  }
  *out = g;
  return AB_OK;
}

extern "C" void ab_graph_destroy(ab_graph *g) {
  if (!g) return;
  cudaSetDevice(g->device);
  for (auto &c : g->ctxs) {
    cudaFree(c.d_list);
    cudaFree(c.d_hash);
    cudaFree(c.d_bits);
    cudaFree(c.d_bits_x);
    cudaFree(c.d_neg);
    cudaFree(c.d_hq);
  cudaFree(c.d_fbits);
  cudaFree(c.d_fbits_x);
    cudaFree(c.d_fbits);
    cudaFree(c.d_fbits_x);
  }
  cudaFree(g->d_ctxs);
  cudaFree(g->e_rng);
  cudaFree(g->x_rng);
  cudaFree(g->deg);
  cudaFree(g->e_arcs);
  cudaFree(g->x_arcs);
  cudaFree(g->final_cost);
  cudaFree(g->d_neg0);
  if (g->stream) cudaStreamDestroy(g->stream);
  delete g;
}

extern "C" int ab_graph_query(const ab_graph *g, int32_t *num_emitting_labels,
                              int32_t *weights_f32, int64_t *device_bytes) {
  if (!g) return fail(AB_ERR_INVALID, "null graph");
  if (num_emitting_labels) *num_emitting_labels = g->L;
  if (weights_f32) *weights_f32 = g->fmt16 ? 1 : 0;
  if (device_bytes) *device_bytes = (int64_t)g->bytes;
  return AB_OK;
}

// ---------------------------------------------------------------- contexts

// Epsilon slack of a weighting of the graph (the kernel's expansion-time
// cutoff, decode_kernel.cuh advance()): S = -min over states s of h(s), where
// h(s) = min(0, cheapest epsilon path leaving s) under the effective weights
// w + discount on boosted arcs (biasing.py:166-171).  An epsilon path lowers a
// token's cost by at most S.  Computed backwards from the negative epsilon arcs
// (Bellman-Ford over reverse epsilon arcs, only states whose h drops below 0
// are visited).  When h has not settled after 64 rounds (a negative epsilon
// cycle, or a longer negative chain) the result bounds paths of at most 64
// arcs only: *rounds_ok = 64 (the kernel then uses it for max_epsilon_expansion
// <= 64 only), else INT_MAX.  neg_bits: Bloom filter of the states with
// h < 0 (decode_kernel.cuh neg_test).  `boosted` = sorted arc ids.
static double eps_slack(ab_graph *g, const std::vector<u32> &boosted, double discount,
                        std::vector<u32> *neg_bits, int *rounds_ok, std::vector<u32> *hq,
                        double *hq_unit, u32 *neg_count) {
  if (!boosted.empty() && discount >= 0.0 && g->xe_neg.size() == 0) {
    // boosting only raises weights: no negative epsilon arc anywhere
    neg_bits->assign(NEG_BLOCK_WORDS, 0u);
    if (neg_count) *neg_count = 0;
    *rounds_ok = INT32_MAX;
    return 0.0;
  }
  auto is_boosted = [&](u32 gid) { return std::binary_search(boosted.begin(), boosted.end(), gid); };
  auto weff = [&](u32 i) { return is_boosted(g->xe_g[i]) ? g->xe_w[i] + discount : g->xe_w[i]; };
  if (g->h_buf.empty()) g->h_buf.assign((size_t)g->num_states, 0.0);
  std::vector<double> &h = g->h_buf;
  std::vector<u32> front, next, touched;
  auto lower = [&](u32 s, double c, std::vector<u32> &out) {
    if (c < h[s]) {
      if (h[s] == 0.0) touched.push_back(s);
      h[s] = c;
      out.push_back(s);
    }
  };
  // negative epsilon arcs: the graph's own (not boosted) and boosted ones below 0
  for (u32 i : g->xe_neg)
    if (weff(i) < 0.0) lower(g->xe_src[i], weff(i), front);
  if (discount < 0.0)
    for (u32 gid : boosted) {
      auto it = std::lower_bound(g->xe_g.begin(), g->xe_g.end(), gid);
      if (it == g->xe_g.end() || *it != gid) continue; // not an epsilon arc
      const u32 i = (u32)(it - g->xe_g.begin());
      if (g->xe_w[i] >= 0.0 && g->xe_w[i] + discount < 0.0) lower(g->xe_src[i], g->xe_w[i] + discount, front);
    }
  int rounds = 0;
  while (!front.empty() && rounds < 64) {
    std::sort(front.begin(), front.end());
    front.erase(std::unique(front.begin(), front.end()), front.end());
    next.clear();
    for (u32 d : front)
      for (u32 k = g->xr_off[d]; k < g->xr_off[d + 1]; ++k) {
        const u32 i = g->xr_arc[k];
        lower(g->xe_src[i], weff(i) + h[d], next);
      }
    front.swap(next);
    ++rounds;
  }
  double lo = 0.0;
  neg_bits->assign(NEG_WORDS, 0u);
  size_t n_neg = 0;
  for (u32 s : touched) lo = std::min(lo, h[s]);
  for (u32 s : touched) n_neg += h[s] < 0.0;
  // too many states for the Bloom filter to stay sparse: 2-bit per-state slack
  const bool dense = hq && n_neg > HQ_MIN_STATES;
  if (dense) {
    hq->assign(((size_t)g->num_states + HQ_PER_WORD - 1) / HQ_PER_WORD, 0u);
    *hq_unit = -lo * (1.0 + 1e-9) / (double)HQ_MAX + 1e-12;
  }
  for (u32 s : touched) {
    if (dense && h[s] < 0.0) { // rounded up: a conservative per-state slack
      const u32 q = (u32)std::min((double)HQ_MAX, std::ceil(-h[s] * (1.0 + 1e-9) / *hq_unit + 1e-9));
      (*hq)[s / HQ_PER_WORD] |= std::max(q, 1u) << ((s % HQ_PER_WORD) * HQ_BITS);
    }
    if (h[s] < 0.0) {
      (*neg_bits)[neg_h1(s) >> 5] |= 1u << (neg_h1(s) & 31);
      (*neg_bits)[neg_h2(s) >> 5] |= 1u << (neg_h2(s) & 31);
    }
    h[s] = 0.0;
  }
  *rounds_ok = front.empty() ? INT32_MAX : 64;
  // every folded size after the full filter (decode_kernel.cuh NEG_MIN_WORDS)
  neg_bits->resize(NEG_BLOCK_WORDS, 0u);
  for (u32 W = NEG_WORDS / 2, at = NEG_WORDS, prev = 0; W >= NEG_MIN_WORDS; prev = at, at += W, W /= 2)
    for (u32 j = 0; j < 32 * W; ++j) {
      const u32 b0 = 2 * j, b1 = 2 * j + 1;
      const u32 *p = neg_bits->data() + prev;
      if (((p[b0 >> 5] >> (b0 & 31)) | (p[b1 >> 5] >> (b1 & 31))) & 1u) (*neg_bits)[at + (j >> 5)] |= 1u << (j & 31);
    }
  if (neg_count) *neg_count = (u32)n_neg;
  // margin for the f64 rounding of path sums (the kernel adds its own for the hint)
  return lo < 0.0 ? -lo * (1.0 + 1e-9) + 1e-9 : 0.0;
}

static int sync_ctx_table(ab_graph *g) {
  std::vector<CtxDesc> h(g->ctxs.size());
  for (size_t i = 0; i < g->ctxs.size(); ++i) {
    const HostCtx &c = g->ctxs[i];
    h[i].discount = c.discount;
    h[i].k = c.live ? c.k : 0;
    h[i].mode = c.mode;
    h[i].words = c.words;
    h[i].lmask = c.list_mask;
    h[i].list = c.d_list;
    h[i].hash = c.d_hash;
    h[i].bits = c.d_bits;
    h[i].bits_x = c.d_bits_x;
    h[i].slack = c.slack;
    h[i].slack_rounds = c.slack_rounds;
    h[i].neg = c.d_neg;
    h[i].hq = c.d_hq;
    h[i].hq_unit = c.hq_unit;
    h[i].fbits = c.d_fbits;
    h[i].fbits_x = c.d_fbits_x;
  }
  if (h.size() > g->d_ctxs_cap) {
    cudaFree(g->d_ctxs);
    g->d_ctxs = nullptr;
    size_t nc = std::max<size_t>(64, h.size() * 2);
    CK(cudaMalloc(&g->d_ctxs, nc * sizeof(CtxDesc)));
    g->d_ctxs_cap = nc;
  }
  if (!h.empty()) CK(cudaMemcpy(g->d_ctxs, h.data(), h.size() * sizeof(CtxDesc), cudaMemcpyHostToDevice));
  return AB_OK;
}

extern "C" int ab_context_register(ab_graph *g, const int64_t *arc_indices, int64_t k,
                                   double discount, int32_t mode, int32_t *handle) {
  if (!g) return fail(AB_ERR_INVALID, "null graph");
  if (!std::isfinite(discount)) return fail(AB_ERR_INVALID, "non-finite discount");
  for (int64_t i = 0; i < k; ++i) {
    if (arc_indices[i] < 0) return fail(AB_ERR_INVALID, "negative arc index");
    if (i && arc_indices[i] <= arc_indices[i - 1])
      return fail(AB_ERR_INVALID, "arc_indices must be strictly increasing");
  }
  CK(cudaSetDevice(g->device));
  // indices outside the graph can never match an expanded arc (biasing.py:108-117)
  std::vector<u32> list;
  list.reserve(k);
  for (int64_t i = 0; i < k; ++i)
    if (arc_indices[i] < g->num_arcs) list.push_back((u32)arc_indices[i]);
  HostCtx c;
  c.live = true;
  c.discount = discount;
  c.k = (u32)list.size();
  // label-closed? (the context is exactly {g : olabel[g] in W} for W = its olabels)
  bool closed = false;
  std::vector<u32> lbits;
  if (!g->ol_count.empty() && !list.empty()) {
    std::vector<int32_t> labs;
    labs.reserve(list.size());
    for (u32 a : list) labs.push_back(g->olabels[a]);
    std::sort(labs.begin(), labs.end());
    labs.erase(std::unique(labs.begin(), labs.end()), labs.end());
    uint64_t cover = 0;
    for (int32_t l : labs) cover += g->ol_count[l];
    if (cover == list.size() && labs.back() < 32 * CTX_SMEM_WORDS) {
      closed = true;
      lbits.assign((size_t)labs.back() / 32 + 1, 0u);
      for (int32_t l : labs) lbits[l >> 5] |= 1u << (l & 31);
    }
  }
  if (mode == AB_CTX_AUTO)
    mode = closed ? AB_CTX_LABELS : (c.k <= LIST_SMEM_MAX ? AB_CTX_LIST : AB_CTX_BITSET);
  if (mode == AB_CTX_LABELS && !closed)
    return fail(AB_ERR_INVALID, "context is not label-closed: AB_CTX_LABELS would change it");
  if (mode != AB_CTX_LIST && mode != AB_CTX_BITSET && mode != AB_CTX_LABELS)
    return fail(AB_ERR_INVALID, "bad context mode %d", mode);
  c.abi_mode = mode;
  std::vector<u32> negb;
  std::vector<u32> hq;
  c.slack = eps_slack(g, list, discount, &negb, &c.slack_rounds, &hq, &c.hq_unit, &c.neg_count);
  if (!hq.empty()) {
    CK(cudaMalloc(&c.d_hq, hq.size() * sizeof(u32)));
    CK(cudaMemcpy(c.d_hq, hq.data(), hq.size() * sizeof(u32), cudaMemcpyHostToDevice));
    // which records lead to such a state, by record position: read next to
    // the record (one coalesced word per 32 records), so only those
    // candidates look their destination's slack up
    const size_t we = (size_t)(g->e_tot + 31) / 32 + 1, wx = (size_t)(g->x_tot + 31) / 32 + 1;
    std::vector<u32> fe(we, 0), fx(wx, 0);
    for (int64_t a = 0; a < g->num_arcs; ++a) {
      const u32 d = g->arc_dst[a];
      if (!hq_get(hq.data(), d)) continue;
      const u32 p = g->arc_pos[a];
      if (p & 0x80000000u) fx[(p & 0x7FFFFFFFu) >> 5] |= 1u << (p & 31);
      else fe[p >> 5] |= 1u << (p & 31);
    }
    CK(cudaMalloc(&c.d_fbits, we * sizeof(u32)));
    CK(cudaMemcpy(c.d_fbits, fe.data(), we * sizeof(u32), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&c.d_fbits_x, wx * sizeof(u32)));
    CK(cudaMemcpy(c.d_fbits_x, fx.data(), wx * sizeof(u32), cudaMemcpyHostToDevice));
  }
  CK(cudaMalloc(&c.d_neg, NEG_BLOCK_WORDS * sizeof(u32)));
  CK(cudaMemcpy(c.d_neg, negb.data(), NEG_BLOCK_WORDS * sizeof(u32), cudaMemcpyHostToDevice));
  c.mode = mode == AB_CTX_LABELS ? CTX_LABELS : mode == AB_CTX_BITSET ? CTX_BITSET : CTX_SLIST;
  { // the ids as a hash set (load <= 1/2, linear probing): one or two loads per lookup
    u32 hs = 2;
    while (hs < 2 * list.size()) hs <<= 1;
    std::vector<u32> set(hs, 0xFFFFFFFFu);
    for (u32 a : list) {
      u32 h = list_slot(a, hs - 1);
      while (set[h] != 0xFFFFFFFFu && set[h] != a) h = (h + 1) & (hs - 1);
      set[h] = a;
    }
    c.list_mask = hs - 1;
    CK(cudaMalloc(&c.d_list, hs * sizeof(u32)));
    CK(cudaMemcpy(c.d_list, set.data(), hs * sizeof(u32), cudaMemcpyHostToDevice));
  }
  if (mode == AB_CTX_LIST && c.k <= LIST_SMEM_MAX) { // shared-memory Bloom filter (else global search only)
    u32 words = 64;
    while (words < c.k) words <<= 1; // 32 bits per arc
    std::vector<u32> bloom(words, 0u);
    for (u32 a : list) {
      const u32 b1 = list_b1(a, 32 * words), b2 = list_b2(a, 32 * words);
      bloom[b1 >> 5] |= 1u << (b1 & 31);
      bloom[b2 >> 5] |= 1u << (b2 & 31);
    }
    c.words = words;
    CK(cudaMalloc(&c.d_hash, words * sizeof(u32)));
    CK(cudaMemcpy(c.d_hash, bloom.data(), words * sizeof(u32), cudaMemcpyHostToDevice));
  }
  if (mode == AB_CTX_BITSET) {
    // one bit per record position of each arc array (biasing.py:108-117 by
    // position instead of arc id: the same set, addressed without the record)
    const size_t we = (size_t)(g->e_tot + 31) / 32 + 1, wx = (size_t)(g->x_tot + 31) / 32 + 1;
    std::vector<u32> be(we, 0), bx(wx, 0);
    for (u32 a : list) {
      const u32 p = g->arc_pos[a];
      if (p & 0x80000000u) bx[(p & 0x7FFFFFFFu) >> 5] |= 1u << (p & 31);
      else be[p >> 5] |= 1u << (p & 31);
    }
    CK(cudaMalloc(&c.d_bits, we * sizeof(u32)));
    CK(cudaMemcpy(c.d_bits, be.data(), we * sizeof(u32), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&c.d_bits_x, wx * sizeof(u32)));
    CK(cudaMemcpy(c.d_bits_x, bx.data(), wx * sizeof(u32), cudaMemcpyHostToDevice));
  } else if (mode == AB_CTX_LABELS) {
    c.words = (u32)lbits.size();
    CK(cudaMalloc(&c.d_bits, lbits.size() * sizeof(u32)));
    CK(cudaMemcpy(c.d_bits, lbits.data(), lbits.size() * sizeof(u32), cudaMemcpyHostToDevice));
  }
  int h = -1;
  for (size_t i = 0; i < g->ctxs.size(); ++i)
    if (!g->ctxs[i].live) {
      h = (int)i;
      break;
    }
  if (h < 0) {
    h = (int)g->ctxs.size();
    g->ctxs.push_back(c);
  } else {
    g->ctxs[h] = c;
  }
  int rc = sync_ctx_table(g);
  if (rc) return rc;
  *handle = h;
  return AB_OK;
}

extern "C" int ab_context_mode(const ab_graph *g, int32_t handle, int32_t *mode) {
  if (!g || handle < 0 || handle >= (int)g->ctxs.size() || !g->ctxs[handle].live)
    return fail(AB_ERR_UNKNOWN_CTX, "unknown context handle %d", handle);
  *mode = g->ctxs[handle].abi_mode;
  return AB_OK;
}

extern "C" int ab_context_slack(const ab_graph *g, int32_t handle, double *slack, int32_t *neg_states) {
  if (!g) return fail(AB_ERR_INVALID, "null graph");
  const u32 *bits = nullptr;
  std::vector<u32> hb(NEG_WORDS);
  if (handle < 0) {
    *slack = g->slack0;
    bits = g->d_neg0;
  } else {
    if (handle >= (int)g->ctxs.size() || !g->ctxs[handle].live)
      return fail(AB_ERR_UNKNOWN_CTX, "unknown context handle %d", handle);
    *slack = g->ctxs[handle].slack;
    bits = g->ctxs[handle].d_neg;
  }
  CK(cudaMemcpy(hb.data(), bits, NEG_WORDS * sizeof(u32), cudaMemcpyDeviceToHost));
  int n = 0;
  for (u32 w : hb) n += __builtin_popcount(w);
  if (handle < 0 ? g->slack0_rounds < INT32_MAX : g->ctxs[handle].slack_rounds < INT32_MAX) n = -n;
  *neg_states = n;
  return AB_OK;
}

extern "C" int ab_context_release(ab_graph *g, int32_t handle) {
  if (!g || handle < 0 || handle >= (int)g->ctxs.size() || !g->ctxs[handle].live)
    return fail(AB_ERR_UNKNOWN_CTX, "unknown context handle %d", handle);
  CK(cudaSetDevice(g->device));
  HostCtx &c = g->ctxs[handle];
  cudaFree(c.d_list);
  cudaFree(c.d_hash);
  cudaFree(c.d_bits);
  cudaFree(c.d_bits_x);
  cudaFree(c.d_neg);
  cudaFree(c.d_hq);
  cudaFree(c.d_fbits);
  cudaFree(c.d_fbits_x);
  c = HostCtx();
  return sync_ctx_table(g);
}

// ----------------------------------------------------------------- decoder

static u32 next_pow2(uint64_t v) {
  u32 p = 16;
  while (p < v) p <<= 1;
  return p;
}

extern "C" int ab_decoder_create(ab_graph *g, const ab_capacity *capin, int32_t max_channels,
                                 ab_decoder **out) {
  *out = nullptr;
  if (!g) return fail(AB_ERR_INVALID, "null graph");
  if (max_channels < 1) return fail(AB_ERR_INVALID, "max_channels must be >= 1");
  CK(cudaSetDevice(g->device));
  ab_capacity cap = capin ? *capin : ab_capacity{};
  ab_decoder *d = new ab_decoder();
  d->g = g;
  d->device = g->device;
  d->max_ch = max_channels;
  d->slot_ctx.assign((size_t)max_channels, -1);
  // Token table: direct (one value per graph state) when it fits the memory
  // budget next to the other per-channel pools, else hashed.  table_slots > 0
  // forces the choice: >= num_states gives a direct table, fewer slots a
  // hashed one.
  const uint64_t S = (uint64_t)g->num_states;
  int64_t ts = cap.table_slots;
  if (ts <= 0) {
    const uint64_t tk = std::min<uint64_t>(S, MAX_TOKENS);
    const uint64_t fl = cap.frontier_rows > 0 ? (uint64_t)cap.frontier_rows : std::max<uint64_t>(65536, 2 * tk);
    const uint64_t ar = cap.arena_records > 0 ? (uint64_t)cap.arena_records : std::max<uint64_t>(1ull << 19, 8 * fl);
    const double per_ch_other = (double)tk * (4 + 8 + 16 + 16) + (double)fl * (4 + 8 + 16 + 16 + 4 + 4 + 8 + 4) +
                                (double)ar * (2 * 8 + 2 * 4.0 / 32);
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    double budget = 0.85 * (double)free_b - (double)max_channels * per_ch_other;
    if (const char *e = getenv("AB_DIRECT_TABLE_GB")) budget = atof(e) * 1e9;
    const double direct = (double)max_channels * (double)S * (2 * sizeof(u64));
    ts = (S <= MAX_TOKENS || direct <= budget) ? (int64_t)S
                                              : (int64_t)std::min<uint64_t>(next_pow2(4 * MAX_TOKENS), next_pow2(S));
  }
  if ((uint64_t)ts >= S) {
    d->hashed = 0;
    d->table_cap = (u32)S;
  } else {
    d->hashed = 1;
    d->table_cap = next_pow2((uint64_t)ts);
    if (d->table_cap > MAX_HASH_SLOTS) {
      delete d;
      return fail(AB_ERR_INVALID, "table_slots too large (max %u)", MAX_HASH_SLOTS);
    }
  }
  d->tok_cap = std::min<u32>(d->table_cap, MAX_TOKENS);
  d->flog_cap = (u32)(cap.frontier_rows > 0 ? cap.frontier_rows
                                            : std::max<uint64_t>(65536, 2ull * d->tok_cap));
  // the arena must hold the live records plus one frame of appends (<= frontier rows)
  d->arena_cap = (u32)(cap.arena_records > 0 ? cap.arena_records
                                             : std::max<uint64_t>(1ull << 19, 8ull * d->flog_cap));
  d->arena_cap = (d->arena_cap + 31) & ~31u;
  if (d->flog_cap > MAX_ROWS) {
    delete d;
    return fail(AB_ERR_INVALID, "frontier_rows too large (max %u)", MAX_ROWS);
  }
  if ((uint64_t)d->arena_cap < 2ull * d->flog_cap) {
    delete d;
    return fail(AB_ERR_INVALID, "arena_records must be at least twice frontier_rows");
  }
  d->path_cap = (u32)(cap.path_words > 0 ? cap.path_words : (1ll << 16));
  d->cap.table_slots = d->table_cap;
  d->cap.frontier_rows = d->flog_cap;
  d->cap.arena_records = d->arena_cap;
  d->cap.path_words = d->path_cap;
  const size_t C = (size_t)max_channels;
  size_t &acc = d->bytes;
  const size_t hslots = d->hashed ? C * d->table_cap : 0, dslots = d->hashed ? 0 : C * d->table_cap;
  if (dmalloc(&d->chans, C, acc) || (hslots && dmalloc(&d->table, hslots, acc)) ||
      (dslots && dmalloc(&d->vals, 2 * dslots, acc)) ||
      dmalloc(&d->tok_state, C * d->tok_cap, acc) || dmalloc(&d->tok_cost, C * d->tok_cap, acc) ||
      dmalloc(&d->tok_info, 2 * C * d->tok_cap, acc) ||
      dmalloc(&d->flog_state, C * d->flog_cap, acc) ||
      dmalloc(&d->flog_ck, C * d->flog_cap, acc) ||
      dmalloc(&d->flog_aux, C * d->flog_cap, acc) || dmalloc(&d->eps_list, C * d->flog_cap, acc) ||

      dmalloc(&d->app_list, C * d->flog_cap, acc) || dmalloc(&d->flog_kill, C * d->flog_cap, acc) ||
      dmalloc(&d->scr_key, C * d->flog_cap, acc) ||
      dmalloc(&d->scr_row, C * d->flog_cap, acc) ||
      dmalloc(&d->arena, 2 * C * d->arena_cap, acc) ||
      dmalloc(&d->gc_bits, C * (d->arena_cap / 32 + 1), acc) ||
      dmalloc(&d->gc_rank, C * (d->arena_cap / 32 + 1), acc) ||
      dmalloc(&d->path_rec, C * d->path_cap, acc) ||
      dmalloc(&d->path_words, C * d->path_cap, acc)) {
    size_t need = acc;
    ab_decoder_destroy(d);
    return fail(AB_ERR_CUDA, "device allocation for %d channels failed (%zu bytes requested)",
                max_channels, need);
  }
  if ((hslots && cudaMemset(d->table, 0, hslots * sizeof(Entry)) != cudaSuccess) ||
      (dslots && cudaMemset(d->vals, 0, dslots * 2 * sizeof(u64)) != cudaSuccess) ||
      cudaMemset(d->chans, 0, C * sizeof(ChanState)) != cudaSuccess ||
      cudaMemset(d->flog_kill, 0, C * d->flog_cap * sizeof(u32)) != cudaSuccess || // (no valid tag)
      cudaEventCreate(&d->ev0) != cudaSuccess || cudaEventCreate(&d->ev1) != cudaSuccess) {
    ab_decoder_destroy(d);
    return fail(AB_ERR_CUDA, "decoder init failed");
  }
  std::vector<ChanState> init(C);
  for (auto &c : init) {
    memset(&c, 0, sizeof(c));
    c.info.status = AB_IDLE;
    c.info.fresh = 1;
    c.info.context = -1;
  }
  if (cudaMemcpy(d->chans, init.data(), C * sizeof(ChanState), cudaMemcpyHostToDevice) !=
      cudaSuccess) {
    ab_decoder_destroy(d);
    return fail(AB_ERR_CUDA, "decoder init copy failed");
  }
  *out = d;
  return AB_OK;
}

extern "C" void ab_decoder_destroy(ab_decoder *d) {
  if (!d) return;
  cudaSetDevice(d->device); // never touches d->g: the graph may already be gone
  void *ptrs[] = {d->chans,     d->table,     d->vals, d->tok_state, d->tok_cost, d->tok_info,
                  d->flog_state, d->flog_ck,  d->flog_aux, d->eps_list, d->app_list,
                  d->flog_kill, d->scr_key,   d->scr_row,   d->arena,     d->path_rec, d->path_words,
                  d->gc_bits,   d->gc_rank,
                  d->d_slots,   d->d_frames,  d->d_sframes, d->d_nhyps,   d->d_errors, d->d_done,
                  d->d_soff,    d->d_wused,   d->d_hyps,    d->d_words,  d->d_packh,
                  d->d_packw,   d->d_packoff, d->d_stage, d->d_infos, d->d_islots};
  for (void *p : ptrs) cudaFree(p);
  if (d->ev0) cudaEventDestroy(d->ev0);
  if (d->ev1) cudaEventDestroy(d->ev1);
  for (auto e : d->ev_copy)
    if (e) cudaEventDestroy(e);
  if (d->copy_stream) cudaStreamDestroy(d->copy_stream);
  delete d;
}

extern "C" int ab_decoder_query(const ab_decoder *d, ab_capacity *cap, int64_t *device_bytes) {
  if (!d) return fail(AB_ERR_INVALID, "null decoder");
  if (cap) *cap = d->cap;
  if (device_bytes) *device_bytes = (int64_t)d->bytes;
  return AB_OK;
}

static int check_slot(ab_decoder *d, int ch) {
  if (!d) return fail(AB_ERR_INVALID, "null decoder");
  if (ch < 0 || ch >= d->max_ch)
    return fail(AB_ERR_INVALID, "channel slot %d out of range [0, %d)", ch, d->max_ch);
  return AB_OK;
}

static int check_ctx(ab_decoder *d, int ctx) {
  if (ctx < 0) return AB_OK;
  if (ctx >= (int)d->g->ctxs.size() || !d->g->ctxs[ctx].live)
    return fail(AB_ERR_UNKNOWN_CTX, "unknown context handle %d", ctx);
  return AB_OK;
}

extern "C" int ab_channel_init(ab_decoder *d, int32_t ch, int32_t context) {
  int rc;
  if ((rc = check_slot(d, ch)) || (rc = check_ctx(d, context))) return rc;
  CK(cudaSetDevice(d->g->device));
  ab_channel_info info;
  memset(&info, 0, sizeof(info));
  info.status = AB_IDLE;
  info.fresh = 1;
  info.context = context;
  d->slot_ctx[ch] = context;
  // the epoch and path fields stay: epochs must never repeat within a slot
  CK(cudaMemcpy(&d->chans[ch].info, &info, sizeof(info), cudaMemcpyHostToDevice));
  int zero[4] = {0, 0, 0, 0}; // path_len, max_depth, arena_half, rec_phys
  CK(cudaMemcpy(&d->chans[ch].path_len, zero, sizeof(zero), cudaMemcpyHostToDevice));
  return AB_OK;
}

extern "C" int ab_channel_get(ab_decoder *d, int32_t ch, ab_channel_info *info) {
  int rc;
  if ((rc = check_slot(d, ch))) return rc;
  CK(cudaSetDevice(d->g->device));
  CK(cudaMemcpy(info, &d->chans[ch].info, sizeof(*info), cudaMemcpyDeviceToHost));
  return AB_OK;
}

extern "C" int ab_channel_put(ab_decoder *d, int32_t ch, const ab_channel_info *info) {
  int rc;
  if ((rc = check_slot(d, ch)) || (rc = check_ctx(d, info->context))) return rc;
  CK(cudaSetDevice(d->g->device));
  CK(cudaMemcpy(&d->chans[ch].info, info, sizeof(*info), cudaMemcpyHostToDevice));
  d->slot_ctx[ch] = info->context;
  return AB_OK;
}

extern "C" int ab_channel_set_context(ab_decoder *d, int32_t ch, int32_t context) {
  int rc;
  if ((rc = check_slot(d, ch)) || (rc = check_ctx(d, context))) return rc;
  ab_channel_info info;
  if ((rc = ab_channel_get(d, ch, &info))) return rc;
  if (info.status != AB_IDLE && info.status != AB_FINISHED)
    return fail(AB_ERR_STATUS, "context switch mid-utterance (status %d)", info.status);
  info.context = context;
  if (info.status == AB_FINISHED) info.status = AB_IDLE;
  return ab_channel_put(d, ch, &info);
}

__global__ void gather_infos(int n, const int *slots, const ChanState *chans,
                             ab_channel_info *out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = chans[slots[i]].info;
}

__global__ void scatter_infos(int n, const int *slots, ChanState *chans,
                              const ab_channel_info *in, int reset_path) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    chans[slots[i]].info = in[i];
    if (reset_path) {
      chans[slots[i]].path_len = 0;
      chans[slots[i]].max_depth = 0;
      chans[slots[i]].arena_half = 0;
      chans[slots[i]].rec_phys = 0;
      chans[slots[i]].prev_cut = INFINITY;
      chans[slots[i]].cut_rise = 0.0;
      chans[slots[i]].best_tok = -1;
    }
  }
}

static int ensure_infos(ab_decoder *d, int n) {
  if ((size_t)n <= d->info_cap) return AB_OK;
  cudaFree(d->d_infos);
  cudaFree(d->d_islots);
  size_t nc = std::max<size_t>(n, 64);
  CK(cudaMalloc(&d->d_infos, nc * sizeof(ab_channel_info)));
  CK(cudaMalloc(&d->d_islots, nc * sizeof(int)));
  d->info_cap = nc;
  return AB_OK;
}

extern "C" int ab_channels_get(ab_decoder *d, int32_t n, const int32_t *slots,
                               ab_channel_info *infos) {
  if (!d || n < 0) return fail(AB_ERR_INVALID, "bad arguments");
  if (n == 0) return AB_OK;
  int rc;
  for (int i = 0; i < n; ++i)
    if ((rc = check_slot(d, slots[i]))) return rc;
  CK(cudaSetDevice(d->g->device));
  if ((rc = ensure_infos(d, n))) return rc;
  cudaStream_t st = d->g->stream;
  CK(cudaMemcpyAsync(d->d_islots, slots, n * sizeof(int), cudaMemcpyHostToDevice, st));
  gather_infos<<<(n + 127) / 128, 128, 0, st>>>(n, d->d_islots, d->chans, d->d_infos);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(infos, d->d_infos, n * sizeof(ab_channel_info), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return AB_OK;
}

static int put_infos(ab_decoder *d, int n, const int32_t *slots, const ab_channel_info *infos,
                     int reset_path) {
  int rc;
  CK(cudaSetDevice(d->g->device));
  if ((rc = ensure_infos(d, n))) return rc;
  for (int i = 0; i < n; ++i) d->slot_ctx[slots[i]] = infos[i].context;
  cudaStream_t st = d->g->stream;
  CK(cudaMemcpyAsync(d->d_islots, slots, n * sizeof(int), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d->d_infos, infos, n * sizeof(ab_channel_info), cudaMemcpyHostToDevice, st));
  scatter_infos<<<(n + 127) / 128, 128, 0, st>>>(n, d->d_islots, d->chans, d->d_infos, reset_path);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  return AB_OK;
}

extern "C" int ab_channels_init(ab_decoder *d, int32_t n, const int32_t *slots,
                                const int32_t *contexts) {
  if (!d || n < 0) return fail(AB_ERR_INVALID, "bad arguments");
  int rc;
  std::vector<ab_channel_info> v(n);
  for (int i = 0; i < n; ++i) {
    if ((rc = check_slot(d, slots[i])) || (rc = check_ctx(d, contexts ? contexts[i] : -1))) return rc;
    memset(&v[i], 0, sizeof(ab_channel_info));
    v[i].status = AB_IDLE;
    v[i].fresh = 1;
    v[i].context = contexts ? contexts[i] : -1;
  }
  return n ? put_infos(d, n, slots, v.data(), 1) : AB_OK;
}

extern "C" int ab_channels_set_context(ab_decoder *d, int32_t n, const int32_t *slots,
                                       const int32_t *contexts) {
  if (!d || n < 0) return fail(AB_ERR_INVALID, "bad arguments");
  if (n == 0) return AB_OK;
  int rc;
  std::vector<ab_channel_info> v(n);
  if ((rc = ab_channels_get(d, n, slots, v.data()))) return rc;
  for (int i = 0; i < n; ++i) {
    if ((rc = check_ctx(d, contexts[i]))) return rc;
    if (v[i].status != AB_IDLE && v[i].status != AB_FINISHED)
      return fail(AB_ERR_STATUS, "channel slot %d: context switch mid-utterance (status %d)",
                  slots[i], v[i].status);
    v[i].context = contexts[i];
    if (v[i].status == AB_FINISHED) v[i].status = AB_IDLE;
  }
  return put_infos(d, n, slots, v.data(), 0);
}

extern "C" int ab_channel_tokens(ab_decoder *d, int32_t ch, int32_t *states, double *costs,
                                 int32_t *hits, int32_t *bps, int32_t cap, int32_t *n) {
  int rc;
  if ((rc = check_slot(d, ch))) return rc;
  ab_channel_info info;
  if ((rc = ab_channel_get(d, ch, &info))) return rc;
  *n = info.num_active;
  int m = std::min(cap, info.num_active);
  if (m <= 0) return AB_OK;
  const size_t base = (size_t)ch * d->tok_cap;
  if (states) {
    CK(cudaMemcpy(states, d->tok_state + base, m * sizeof(u32), cudaMemcpyDeviceToHost));
    for (int i = 0; i < m; ++i) states[i] &= (int32_t)ROW_STATE; // the device word keeps degree codes
  }
  if (costs) CK(cudaMemcpy(costs, d->tok_cost + base, m * sizeof(double), cudaMemcpyDeviceToHost));
  if (hits || bps) {
    ChanState cs;
    CK(cudaMemcpy(&cs, d->chans + ch, sizeof(ChanState), cudaMemcpyDeviceToHost));
    const size_t tbase = (2 * (size_t)ch + (cs.tok_half & 1u)) * d->tok_cap;
    std::vector<TokInfo> ti(m);
    CK(cudaMemcpy(ti.data(), d->tok_info + tbase, m * sizeof(TokInfo), cudaMemcpyDeviceToHost));
    for (int i = 0; i < m; ++i) {
      if (hits) hits[i] = ti[i].hits;
      if (bps) bps[i] = ti[i].bp;
    }
  }
  return AB_OK;
}

// ------------------------------------------------------------------ launch

template <typename T> static int grow(T **p, size_t &cap, size_t need, size_t &acc) {
  if (need <= cap) return AB_OK;
  cudaFree(*p);
  *p = nullptr;
  size_t nc = std::max(need, cap * 2);
  if (cudaMalloc((void **)p, nc * sizeof(T)) != cudaSuccess) {
    cap = 0;
    return fail(AB_ERR_CUDA, "device allocation of %zu bytes failed", nc * sizeof(T));
  }
  acc += (nc - cap) * sizeof(T);
  cap = nc;
  return AB_OK;
}

static int ensure_batch(ab_decoder *d, size_t n) {
  if (n <= d->batch_cap) return AB_OK;
  cudaFree(d->d_slots);
  cudaFree(d->d_frames);
  cudaFree(d->d_sframes);
  cudaFree(d->d_nhyps);
  cudaFree(d->d_errors);
  cudaFree(d->d_done);
  cudaFree(d->d_soff);
  cudaFree(d->d_wused);
  cudaFree(d->d_packoff);
  size_t nc = std::max<size_t>(n, 64);
  CK(cudaMalloc(&d->d_slots, nc * sizeof(int)));
  CK(cudaMalloc(&d->d_frames, nc * sizeof(int)));
  CK(cudaMalloc(&d->d_sframes, nc * sizeof(int)));
  CK(cudaMalloc(&d->d_nhyps, nc * sizeof(int)));
  CK(cudaMalloc(&d->d_errors, nc * sizeof(int)));
  CK(cudaMalloc(&d->d_done, nc * sizeof(int)));
  CK(cudaMalloc(&d->d_soff, nc * sizeof(long long)));
  CK(cudaMalloc(&d->d_wused, nc * sizeof(long long)));
  CK(cudaMalloc(&d->d_packoff, 2 * nc * sizeof(long long)));
  d->batch_cap = nc;
  return AB_OK;
}

// Environment knobs read once (ab_reload_env re-reads them): the cutoff
// hint's minimum rise per frame and extra margin (decode_kernel.cuh advance()).
struct Knobs {
  bool loaded = false;
  double hint_min = 1.0, hint_extra = 0.25, hint_warm = 0.0;
  int hint_warm_frames = 0;
};
static Knobs &g_knobs() {
  static Knobs k;
  if (!k.loaded) {
    const char *a = getenv("AB_CUT_HINT_MIN"), *b = getenv("AB_CUT_HINT_EXTRA");
    k.hint_min = a ? atof(a) : 1.0;
    k.hint_extra = b ? atof(b) : 0.25;
    const char *c = getenv("AB_CUT_HINT_WARM"), *d = getenv("AB_CUT_HINT_WARM_FRAMES");
    k.hint_warm = c ? atof(c) : 0.0;
    k.hint_warm_frames = d ? atoi(d) : 0;
    k.loaded = true;
  }
  return k;
}

extern "C" void ab_reload_env(void) { g_knobs().loaded = false; }

static void fill_params(ab_decoder *d, DecodeParams &P) {
  ab_graph *g = d->g;
  memset(&P, 0, sizeof(P));
#ifdef AB_PROFILE
  static unsigned long long *prof = nullptr;
  if (!prof && cudaMalloc(&prof, PF_N * sizeof(unsigned long long)) == cudaSuccess)
    cudaMemset(prof, 0, PF_N * sizeof(unsigned long long));
  P.prof = prof;
#endif
  P.e_rng = g->e_rng;
  P.deg = g->deg;
  P.exact = 1; // the expansion-time cutoff is per decode call (ab_config.flags)
  P.slack0 = g->slack0;
  P.slack0_rounds = g->slack0_rounds;
  P.neg0 = g->d_neg0;
  P.hint_min = g_knobs().hint_min;
  P.hint_extra = g_knobs().hint_extra;
  P.hint_warm = g_knobs().hint_warm;
  P.hint_warm_frames = g_knobs().hint_warm_frames;
  P.e_arcs = g->e_arcs;
  P.x_rng = g->x_rng;
  P.x_arcs = g->x_arcs;
  P.final_cost = g->final_cost;
  P.start = g->start;
  P.num_states = g->num_states;
  P.L = g->L;
  P.ctxs = g->d_ctxs;
  P.num_ctxs = (int)g->ctxs.size();
  P.chans = d->chans;
  P.table = d->table;
  P.vals = d->vals;
  P.table_cap = d->table_cap;
  P.table_mask = d->table_cap - 1;
  int lg = 0;
  while ((1u << lg) < d->table_cap) ++lg;
  P.hash_shift = 32 - lg;
  P.hashed = d->hashed;
  P.tok_state = d->tok_state;
  P.tok_cost = d->tok_cost;
  P.tok_info = d->tok_info;
  P.tok_cap = d->tok_cap;
  P.flog_state = d->flog_state;
  P.flog_ck = d->flog_ck;
  P.final_chunk = 1;
  P.flog_aux = d->flog_aux;
  P.eps_list = d->eps_list;
  P.flog_cap = d->flog_cap;
  P.app_list = d->app_list;
  P.flog_kill = d->flog_kill;
  P.scr_key = d->scr_key;
  P.scr_row = d->scr_row;
  P.arena = d->arena;
  P.arena_cap = d->arena_cap;
  P.gc_bits = d->gc_bits;
  P.gc_rank = d->gc_rank;
  P.path_rec = d->path_rec;
  P.path_words = d->path_words;
  P.path_cap = d->path_cap;
}

#ifndef AB_STAGE_CHUNKS
#define AB_STAGE_FIRST_DIV 32 // host scores: the first chunk is 1/32 of the call's frames
#define AB_STAGE_GROWTH 6     // and each next one up to 6x the previous (copy/decode overlap)
#endif

static size_t dyn_smem_max() { return (CTX_SMEM_WORDS + NEG_WORDS) * sizeof(u32) + SCORE_SMEM_MAX_BYTES; }

// CTA size per batch: few channels get more threads each (a channel's frame
// is one CTA's work), many channels fill the SMs with 256-thread CTAs.
static int pick_block(int n) {
  const char *env = getenv("AB_BLOCK");
  if (env) {
    int b = atoi(env);
    if (b == 256 || b == 512 || b == 1024) return b;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms < 1) sms = 1;
  }
  if (n <= sms) return 1024;
  if (n <= 2 * sms) return 512;
  return 256;
}

// Persistent grid: at most one wave of resident CTAs, and the same number of
// channels for every CTA (n = waves * grid, or within one of it).
template <int BLOCK, typename F, typename S>
static cudaError_t launch_decode(const DecodeParams &P, int n, size_t smem, cudaStream_t st) {
  static int per_sm = -1, sms = 0;
  static size_t attr_set = 0;
  if (smem > attr_set) {
    // static tiles + dynamic (context, score row[, token table]) exceed the 48 KB default
    const size_t want = std::max(dyn_smem_max(), smem);
    cudaFuncSetAttribute(decode_kernel<BLOCK, F, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want);
    attr_set = want;
  }
  if (per_sm < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_kernel<BLOCK, F, S>, BLOCK,
                                                      smem) != cudaSuccess || per_sm < 1)
      per_sm = 1;
  }
  int resident = std::max(1, per_sm * sms);
  const char *env = getenv("AB_GRID");
  if (env && atoi(env) > 0) resident = atoi(env);
  const int waves = (n + resident - 1) / resident;
  const int grid = (n + waves - 1) / waves;
  if (getenv("AB_VERBOSE")) {
    static int said = 0;
    if (said++ < 4) {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, decode_kernel<BLOCK, F, S>);
      fprintf(stderr, "[arcboost] decode_kernel<%d>: %d CTAs/SM, grid %d, static smem %zu, dynamic %zu, regs %d\n",
              BLOCK, per_sm, grid, (size_t)fa.sharedSizeBytes, smem, fa.numRegs);
    }
  }
  decode_kernel<BLOCK, F, S><<<grid, BLOCK, smem, st>>>(P);
  return cudaGetLastError();
}

// One channel per thread-block cluster of CL CTAs (1024 threads, one per SM),
// the small graph's table split across the cluster's shared memory: C1 / C2,
// where one CTA per channel would leave most SMs idle.
template <int CL>
static cudaError_t launch_decode_cluster(const DecodeParams &P, int n, size_t smem, cudaStream_t st) {
  auto kern = decode_kernel<1024, Fmt16SC<CL>, float>;
  static size_t attr_set = 0;
  static int sms = 0;
  if (smem > attr_set) {
    const size_t want = std::max(dyn_smem_max(), smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want);
    if (CL > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr_set = want;
  }
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int max_clusters = std::max(1, sms / CL);
  const int waves = (n + max_clusters - 1) / max_clusters;
  const int nclu = (n + waves - 1) / waves;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nclu * CL), 1, 1);
  cfg.blockDim = dim3(1024, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (getenv("AB_VERBOSE")) {
    static int said = 0;
    if (said++ < 4) fprintf(stderr, "[arcboost] decode_kernel<1024, cluster %d>: %d clusters, dynamic %zu\n", CL, nclu, smem);
  }
  return cudaLaunchKernelEx(&cfg, kern, P);
}

// CTAs per channel for n channels of a small graph (its table in shared
// memory): the largest cluster (8 / 4 / 2) with n clusters resident at once;
// 1 = no cluster.  AB_CLUSTER overrides (1 disables).
static int pick_cluster(int n) {
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (const char *e = getenv("AB_CLUSTER")) {
    const int c = atoi(e);
    return (c == 2 || c == 4 || c == 8 || c == 16) ? c : 1;
  }
  for (int c = 8; c >= 2; c /= 2)
    if ((long long)n * c <= sms) return c;
  return 1;
}

// Whether a channel's direct token table (table_cap 16-byte values) fits in
// shared memory next to the 1024-thread kernel's static tiles and the dynamic
// context / score-row area (`smem`): then the table's loads and CAS-128s stay
// on the SM (small graphs: C1 / C2's 10k states = 160 KB).
template <typename S> static bool smem_table_fits(size_t smem, size_t table_cap) {
  static int optin = -1;
  static size_t stat = 0;
  if (optin < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, decode_kernel<1024, Fmt16S, S>) != cudaSuccess ||
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) {
      (void)cudaGetLastError();
      optin = 0;
    }
    stat = fa.sharedSizeBytes;
  }
  if (getenv("AB_NO_SMEM_TABLE")) return false;
  return stat + smem + table_cap * 16 <= (size_t)optin;
}

template <typename F, typename S>
static cudaError_t launch_decode_b(int block, const DecodeParams &P, int grid, size_t smem,
                                   cudaStream_t st) {
#ifdef AB_ONLY_256 // experiment builds whose tiles do not fit the larger CTAs
  (void)block;
  return launch_decode<256, F, S>(P, grid, smem, st);
#else
  switch (block) {
  case 512: return launch_decode<512, F, S>(P, grid, smem, st);
  case 1024: return launch_decode<1024, F, S>(P, grid, smem, st);
  default: return launch_decode<256, F, S>(P, grid, smem, st);
  }
#endif
}

template <int BLOCK, typename F, typename S>
static cudaError_t launch_hyp(const DecodeParams &P, int which, size_t smem, cudaStream_t st) {
  hyp_kernel<BLOCK, F, S><<<1, BLOCK, smem, st>>>(P, which);
  return cudaGetLastError();
}

// Packs the per-channel hypothesis rows and word regions into contiguous
// buffers (one D2H each); words_off is rewritten to the packed offset.
__global__ void pack_kernel(int n, const int *n_hyps, const long long *wused, const DevHyp *hyps,
                            int hyp_stride, const int *words, long long words_stride,
                            DevHyp *out_h, int *out_w, long long *offs) {
  const int b = blockIdx.x;
  __shared__ long long sh_h, sh_w;
  if (threadIdx.x == 0) {
    sh_h = 0;
    sh_w = 0;
  }
  __syncthreads();
  long long ph = 0, pw = 0;
  for (int c = threadIdx.x; c < b; c += blockDim.x) {
    ph += n_hyps[c];
    pw += wused[c];
  }
  atomicAdd((unsigned long long *)&sh_h, (unsigned long long)ph);
  atomicAdd((unsigned long long *)&sh_w, (unsigned long long)pw);
  __syncthreads();
  const long long hb = sh_h, wb = sh_w;
  const int nh = n_hyps[b];
  const long long nw = wused[b];
  for (int i = threadIdx.x; i < nh; i += blockDim.x) {
    DevHyp h = hyps[(size_t)b * hyp_stride + i];
    h.words_off = wb + (h.words_off - (long long)b * words_stride);
    out_h[hb + i] = h;
  }
  for (long long i = threadIdx.x; i < nw; i += blockDim.x)
    out_w[wb + i] = words[(size_t)b * words_stride + i];
  if (threadIdx.x == 0) {
    offs[2 * b] = hb;
    offs[2 * b + 1] = wb;
  }
}

// Dynamic shared memory of a launch: [context words | score row | neg Bloom
// filter | (small graphs) token table].  The context area holds the largest
// shared-memory context of the launch's channels (LABELS bitmap words or LIST
// arcs, <= CTX_SMEM_WORDS); the Bloom filter is there only when one of them
// (or the unbiased graph) has an epsilon slack.  Shared memory not taken is
// L1 cache for the arc records and token lists.
static void launch_smem_layout(ab_decoder *d, const int32_t *slots, int n, DecodeParams &P) {
  const ab_graph *g = d->g;
  u32 words = 0;
  bool neg = false;
  u32 flagged = 0;
  for (int i = 0; i < n; ++i) {
    const int h = d->slot_ctx[slots[i]];
    const bool live = h >= 0 && h < (int)g->ctxs.size() && g->ctxs[h].live && g->ctxs[h].k;
    if (!live) {
      if (g->slack0 > 0.0) neg = true, flagged = std::max(flagged, g->neg0_count);
      continue;
    }
    const HostCtx &c = g->ctxs[h];
    if (c.mode == CTX_LABELS) words = std::max(words, c.words);
    else if (c.mode == CTX_SLIST && c.words) words = std::max(words, c.words); // its Bloom filter
    if (c.slack > 0.0 && !c.d_hq) neg = true, flagged = std::max(flagged, c.neg_count);
  }
  P.ctx_words_cap = (words + 3) & ~3u; // keeps the score row 16-byte aligned
  u32 W = NEG_MIN_WORDS; // ~8 filter bits per flagged state
  while (W < NEG_WORDS && 32ull * W < 8ull * flagged) W *= 2;
  P.neg_words = neg ? W : 0u;
}

static size_t dyn_smem(int L, bool s64, DecodeParams &P) {
  size_t row = (size_t)L * (s64 ? 8 : 4);
  P.row_in_smem = row <= (size_t)SCORE_SMEM_MAX_BYTES && !getenv("AB_ROW_GLOBAL");
  row = P.row_in_smem ? (row + 15) / 16 * 16 : 0;
  return (size_t)P.ctx_words_cap * sizeof(u32) + row + (size_t)P.neg_words * sizeof(u32);
}

extern "C" int ab_decode(ab_decoder *d, const ab_decode_args *a) {
  if (!d || !a) return fail(AB_ERR_INVALID, "null argument");
  ab_graph *g = d->g;
  const int n = a->n;
  if (n < 0) return fail(AB_ERR_INVALID, "negative batch size");
  d->res_nhyps.assign(n, 0);
  d->res_err.assign(n, 0);
  d->res_hyps.assign(n, {});
  d->res_words.assign(n, {});
  d->last_ms = 0.f;
  d->last_launches = 0;
  if (n == 0) return AB_OK;
  if (a->width != g->L)
    return fail(AB_ERR_WIDTH, "frame width %d does not match the graph's emitting-label count %d",
                a->width, g->L);
  if (a->scores_dtype != AB_F32 && a->scores_dtype != AB_F64)
    return fail(AB_ERR_INVALID, "scores_dtype must be AB_F32 or AB_F64");
  const ab_config &cf = a->config;
  if (!(cf.beam > 0)) return fail(AB_ERR_INVALID, "beam must be positive");
  if (cf.max_active < 1) return fail(AB_ERR_INVALID, "max_active must be >= 1");
  if (cf.partial_every < 1) return fail(AB_ERR_INVALID, "partial_every must be >= 1");
  // max_epsilon_expansion: any value (a round without applications ends the
  // closure; negative = no rounds, decoder.py:263)
  std::vector<int> slots(a->channels, a->channels + n), frames(a->frames, a->frames + n);
  std::vector<long long> soff(a->score_offsets, a->score_offsets + n);
  int64_t maxT = 0, rows = 0;
  for (int i = 0; i < n; ++i) {
    int rc;
    if ((rc = check_slot(d, slots[i]))) return rc;
    if (frames[i] < 0) return fail(AB_ERR_INVALID, "negative frame count");
    maxT = std::max<int64_t>(maxT, frames[i]);
    rows = std::max<int64_t>(rows, (soff[i] / std::max(1, g->L)) + frames[i]);
  }
  {
    std::vector<int> s2 = slots;
    std::sort(s2.begin(), s2.end());
    if (std::adjacent_find(s2.begin(), s2.end()) != s2.end())
      return fail(AB_ERR_INVALID, "a channel appears twice in one batch");
  }
  CK(cudaSetDevice(g->device));
  (void)cudaGetLastError(); // drop stale non-sticky errors of unrelated earlier calls
  cudaStream_t st = a->stream ? (cudaStream_t)a->stream : g->stream;
  const bool s64 = a->scores_dtype == AB_F64;
  const size_t esz = s64 ? 8 : 4;
  (void)rows;
  int rc;
  // Host scores (the end-to-end path): frames [cb[c], cb[c + 1]) of every
  // channel are staged chunk by chunk into two device buffers on a copy
  // stream; the copy of chunk c + 1 overlaps the decode of chunk c.  Utterances continue
  // across chunks; only the last chunk finalizes (decoder.py:498-501).
  const bool host = !a->scores_on_device;
  // chunk c holds frames [cb[c], cb[c + 1]): a short first chunk (its copy is
  // the only one not under a decode), then each up to AB_STAGE_GROWTH times
  // the previous (a frame of every channel decodes ~7x slower than it copies)
  std::vector<int64_t> cb{0};
  if (host && maxT > 0) {
    int64_t len = std::max<int64_t>(1, (maxT + AB_STAGE_FIRST_DIV - 1) / AB_STAGE_FIRST_DIV);
    while (cb.back() < maxT) {
      cb.push_back(std::min<int64_t>(maxT, cb.back() + len));
      len *= AB_STAGE_GROWTH;
    }
  } else {
    cb.push_back(maxT);
  }
  const int K = (int)cb.size() - 1;
  int64_t Tc = 0; // the longest chunk: the staging buffers' rows per channel
  for (int c = 0; c < K; ++c) Tc = std::max<int64_t>(Tc, cb[c + 1] - cb[c]);
  const size_t rowb = (size_t)g->L * esz;
  const size_t bufsz = host ? (size_t)n * (size_t)Tc * rowb : 0;
  if (host) {
    if ((rc = grow((unsigned char **)&d->d_stage, d->stage_cap, 2 * std::max<size_t>(bufsz, 1), d->bytes)))
      return rc;
    if (!d->copy_stream) CK(cudaStreamCreateWithFlags(&d->copy_stream, cudaStreamNonBlocking));
    for (auto &e : d->ev_copy)
      if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  long long stride = n > 1 ? soff[1] - soff[0] : 0;
  bool uniform = true;
  for (int i = 1; i < n && uniform; ++i) uniform = soff[i] - soff[i - 1] == stride;
  auto stage = [&](int c) -> int {
    unsigned char *dst = (unsigned char *)d->d_stage + (size_t)(c & 1) * bufsz;
    const unsigned char *src = (const unsigned char *)a->scores;
    const int64_t f0 = cb[c], tc = cb[c + 1] - cb[c];
    // one 2D copy when the channels' rows are equally strided and disjoint
    bool full = uniform && stride >= tc * (int64_t)g->L;
    for (int i = 0; i < n && full; ++i) full = frames[i] - f0 >= tc;
    if (full && n > 0) {
      CK(cudaMemcpy2DAsync(dst, Tc * rowb, src + ((size_t)soff[0] + (size_t)f0 * g->L) * esz,
                           (size_t)stride * esz, tc * rowb, n, cudaMemcpyHostToDevice, d->copy_stream));
    } else {
      for (int i = 0; i < n; ++i) {
        const int64_t fr = std::min<int64_t>(std::max<int64_t>(frames[i] - f0, 0), tc);
        if (fr > 0)
          CK(cudaMemcpyAsync(dst + (size_t)i * Tc * rowb, src + ((size_t)soff[i] + (size_t)f0 * g->L) * esz,
                             (size_t)fr * rowb, cudaMemcpyHostToDevice, d->copy_stream));
      }
    }
    CK(cudaEventRecord(d->ev_copy[c & 1], d->copy_stream));
    return AB_OK;
  };
  if ((rc = ensure_batch(d, n))) return rc;
  const int stream_mode = a->mode == AB_MODE_STREAM;
  const int hyp_stride = stream_mode ? 2 * (int)std::min<int64_t>(maxT, 1 << 20) + 2 : 1;
  const long long words_stride = stream_mode ? 2ll * d->path_cap + 1024 : 1;
  if ((rc = grow(&d->d_hyps, d->hyps_cap, (size_t)n * hyp_stride, d->bytes)) ||
      (rc = grow(&d->d_words, d->words_cap, (size_t)n * words_stride, d->bytes)))
    return rc;
  DecodeParams P;
  fill_params(d, P);
  P.scores = a->scores;
  P.mode = a->mode;
  P.beam = cf.beam;
  P.max_active = cf.max_active;
  P.max_eps = cf.max_epsilon_expansion;
  P.partial_every = cf.partial_every;
  P.endpoint_silence_frames = cf.endpoint_silence_frames;
  P.silence_ilabel = cf.silence_ilabel;
  P.exact = (cf.flags & AB_CFG_EXACT) ? 1 : 0;
  P.hyps = d->d_hyps;
  P.hyp_stride = hyp_stride;
  P.n_hyps = d->d_nhyps;
  P.errors = d->d_errors;
  P.frames_done = d->d_done;
  P.words = d->d_words;
  P.words_stride = words_stride;
  P.words_used = d->d_wused;
  P.slots = d->d_slots;
  P.frames = d->d_frames;
  P.stream_frames = d->d_sframes;
  P.score_off = d->d_soff;
  launch_smem_layout(d, slots.data(), n, P);
  const size_t smem = dyn_smem(g->L, s64, P);
  std::vector<int> act;
  std::vector<int> remaining(n);
  std::vector<long long> cur_off(n);
  std::vector<int> hn, he, hd;
  std::vector<long long> hw, hoffs;
  std::vector<DevHyp> ph;
  std::vector<int> pw;
  float total_ms = 0.f;
  if (host && (rc = stage(0))) return rc;
  for (int c = 0; c < K; ++c) {
  const int64_t f0 = cb[c], tc = cb[c + 1] - cb[c];
  const bool last = c == K - 1;
  P.final_chunk = last ? 1 : 0;
  if (host) {
    CK(cudaStreamWaitEvent(st, d->ev_copy[c & 1], 0));
    P.scores = (const unsigned char *)d->d_stage + (size_t)(c & 1) * bufsz;
  }
  // active set: channels with frames in this chunk (every channel in the last
  // chunk: a stream ends with its final hypothesis)
  act.clear();
  for (int i = 0; i < n; ++i) {
    if (d->res_err[i]) continue;
    const int64_t fr = host ? std::min<int64_t>(std::max<int64_t>(frames[i] - f0, 0), tc) : frames[i];
    if (fr > 0 || last) act.push_back(i);
    remaining[i] = (int)fr;
    cur_off[i] = host ? (long long)i * Tc * g->L : soff[i];
  }
  bool staged_next = !host || last;
  while (!act.empty()) {
    const int m = (int)act.size();
    std::vector<int> ls(m), lf(m), lt(m);
    std::vector<long long> lo(m);
    for (int j = 0; j < m; ++j) {
      ls[j] = slots[act[j]];
      lf[j] = remaining[act[j]];
      lt[j] = frames[act[j]];
      lo[j] = cur_off[act[j]];
    }
    CK(cudaMemcpyAsync(d->d_sframes, lt.data(), m * sizeof(int), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d->d_slots, ls.data(), m * sizeof(int), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d->d_frames, lf.data(), m * sizeof(int), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d->d_soff, lo.data(), m * sizeof(long long), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(d->d_wused, 0, m * sizeof(long long), st));
    P.n = m;
    const int block = pick_block(m);
    CK(cudaEventRecord(d->ev0, st));
    cudaError_t le;
#ifdef AB_BENCH_ONLY
    // experiment builds (scripts/build_variants.sh): only the C3 bench path
    if (!(g->fmt16 && !s64)) return fail(AB_ERR_INVALID, "AB_BENCH_ONLY build");
    le = d->hashed ? launch_decode_b<Fmt16<true>, float>(block, P, m, smem, st)
                   : launch_decode_b<Fmt16<false>, float>(block, P, m, smem, st);
#else
    if (d->hashed) {
      if (g->fmt16) le = s64 ? launch_decode_b<Fmt16<true>, double>(block, P, m, smem, st)
                             : launch_decode_b<Fmt16<true>, float>(block, P, m, smem, st);
      else le = s64 ? launch_decode_b<Fmt24<true>, double>(block, P, m, smem, st)
                    : launch_decode_b<Fmt24<true>, float>(block, P, m, smem, st);
    } else {
      const int clu = (g->fmt16 && block == 1024 && !s64) ? pick_cluster(m) : 1;
      const size_t part = ((size_t)P.table_cap + clu - 1) / clu * 16; // a cluster CTA's table share
      const bool use_clu = clu > 1 && smem_table_fits<float>(smem, (size_t)P.table_cap / clu + 1);
      if (use_clu)
        le = clu == 16 ? launch_decode_cluster<16>(P, m, smem + part, st)
           : clu == 8 ? launch_decode_cluster<8>(P, m, smem + part, st)
           : clu == 4 ? launch_decode_cluster<4>(P, m, smem + part, st)
                      : launch_decode_cluster<2>(P, m, smem + part, st);
      else if (g->fmt16 && block == 1024 && (s64 ? smem_table_fits<double>(smem, P.table_cap)
                                                 : smem_table_fits<float>(smem, P.table_cap)))
        le = s64 ? launch_decode<1024, Fmt16S, double>(P, m, smem + (size_t)P.table_cap * 16, st)
                 : launch_decode<1024, Fmt16S, float>(P, m, smem + (size_t)P.table_cap * 16, st);
      else if (g->fmt16) le = s64 ? launch_decode_b<Fmt16<false>, double>(block, P, m, smem, st)
                                  : launch_decode_b<Fmt16<false>, float>(block, P, m, smem, st);
      else le = s64 ? launch_decode_b<Fmt24<false>, double>(block, P, m, smem, st)
                    : launch_decode_b<Fmt24<false>, float>(block, P, m, smem, st);
    }
#endif
    if (le != cudaSuccess) return fail(AB_ERR_CUDA, "decode launch: %s", cudaGetErrorString(le));
    d->last_launches += 1;
    CK(cudaEventRecord(d->ev1, st));
    if (!staged_next) { // next chunk's copy runs under this launch
      if ((rc = stage(c + 1))) return rc;
      staged_next = true;
    }
    // pack + read back
    hn.resize(m);
    he.resize(m);
    hd.resize(m);
    hw.resize(m);
    CK(cudaMemcpyAsync(hn.data(), d->d_nhyps, m * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hw.data(), d->d_wused, m * sizeof(long long), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, d->ev0, d->ev1);
    total_ms += ms;
    long long th = 0, tw = 0;
    for (int j = 0; j < m; ++j) {
      th += hn[j];
      tw += hw[j];
    }
    if ((rc = grow(&d->d_packh, d->packh_cap, (size_t)std::max<long long>(th, 1), d->bytes)) ||
        (rc = grow(&d->d_packw, d->packw_cap, (size_t)std::max<long long>(tw, 1), d->bytes)))
      return rc;
    pack_kernel<<<m, 128, 0, st>>>(m, d->d_nhyps, d->d_wused, d->d_hyps, hyp_stride, d->d_words,
                                   words_stride, d->d_packh, d->d_packw, d->d_packoff);
    CK(cudaGetLastError());
    d->last_launches += 1;
    ph.resize(std::max<long long>(th, 1));
    pw.resize(std::max<long long>(tw, 1));
    hoffs.resize(2 * m);
    if (th) CK(cudaMemcpyAsync(ph.data(), d->d_packh, th * sizeof(DevHyp), cudaMemcpyDeviceToHost, st));
    if (tw) CK(cudaMemcpyAsync(pw.data(), d->d_packw, tw * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hoffs.data(), d->d_packoff, 2 * m * sizeof(long long), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(he.data(), d->d_errors, m * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hd.data(), d->d_done, m * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::vector<int> next;
    for (int j = 0; j < m; ++j) {
      const int i = act[j];
      auto &H = d->res_hyps[i];
      auto &Wv = d->res_words[i];
      const long long hb = hoffs[2 * j], wb = hoffs[2 * j + 1];
      for (int q = 0; q < hn[j]; ++q) {
        const DevHyp &x = ph[hb + q];
        ab_hyp y;
        y.cost = x.cost;
        y.frame = x.frame;
        y.kind = x.kind;
        y.fallback = x.fallback;
        y.hits = x.hits;
        y.shared = x.shared;
        y.n_words = x.n_words;
        y.pad_ = 0;
        y.words_off = (int64_t)Wv.size() + (x.words_off - wb);
        H.push_back(y);
      }
      Wv.insert(Wv.end(), pw.begin() + wb, pw.begin() + wb + hw[j]);
      d->res_nhyps[i] += hn[j];
      if (he[j]) {
        d->res_err[i] = he[j];
        continue;
      }
      remaining[i] -= hd[j];
      cur_off[i] += (long long)hd[j] * g->L;
      if (remaining[i] > 0) next.push_back(i);
    }
    act.swap(next);
  }
  }
  d->last_ms = total_ms;
#ifdef AB_PROFILE
  {
    unsigned long long pr[PF_N];
    cudaMemcpy(pr, P.prof, sizeof(pr), cudaMemcpyDeviceToHost);
    static const char *names[PF_N] = {"start", "row", "emit_x", "emit_s", "eps_x", "eps_s",
                                      "prune_scan", "prune_sel", "prune_out", "hyp", "gc", "rounds",
                                      "epoch", "emit_bar", "eps_bar", "adv_bar", "walk", "nhyp", "xlist", "xcand", "xrelax", "phist", "prows", "nsel", "nmem", "npass"};
    fprintf(stderr, "AB_PROFILE");
    for (int q = 0; q < 26; ++q) fprintf(stderr, " %s=%llu", names[q], pr[q]);
    fprintf(stderr, "\n");
    cudaMemset(P.prof, 0, sizeof(pr));
  }
#endif
  return AB_OK;
}

extern "C" int ab_read_results(ab_decoder *d, int32_t *n_hyps, int32_t *errors, ab_hyp *hyps,
                               int32_t hyp_stride, int32_t *words, int64_t words_cap,
                               int64_t *words_used) {
  if (!d) return fail(AB_ERR_INVALID, "null decoder");
  const int n = (int)d->res_nhyps.size();
  int64_t wpos = 0;
  for (int i = 0; i < n; ++i) {
    if (n_hyps) n_hyps[i] = d->res_nhyps[i];
    if (errors) errors[i] = d->res_err[i];
    wpos += (int64_t)d->res_words[i].size();
  }
  if (words_used) *words_used = wpos;
  if (!hyps && !words) return AB_OK;
  if (words && wpos > words_cap) return fail(AB_ERR_CAPACITY, "words buffer too small (%lld)", (long long)wpos);
  int64_t wbase = 0;
  for (int i = 0; i < n; ++i) {
    const auto &H = d->res_hyps[i];
    if (hyps) {
      if ((int)H.size() > hyp_stride) return fail(AB_ERR_CAPACITY, "hyp_stride too small");
      for (size_t q = 0; q < H.size(); ++q) {
        ab_hyp y = H[q];
        y.words_off += wbase;
        hyps[(size_t)i * hyp_stride + q] = y;
      }
    }
    if (words && !d->res_words[i].empty())
      memcpy(words + wbase, d->res_words[i].data(), d->res_words[i].size() * sizeof(int32_t));
    wbase += (int64_t)d->res_words[i].size();
  }
  return AB_OK;
}

static int one_hyp(ab_decoder *d, int32_t ch, int which, ab_hyp *hyp, int32_t *words,
                   int32_t words_cap) {
  int rc;
  if ((rc = check_slot(d, ch))) return rc;
  ab_graph *g = d->g;
  CK(cudaSetDevice(g->device));
  if ((rc = ensure_batch(d, 1))) return rc;
  const long long words_stride = std::max<long long>(d->path_cap, 1);
  if ((rc = grow(&d->d_hyps, d->hyps_cap, 1, d->bytes)) ||
      (rc = grow(&d->d_words, d->words_cap, (size_t)words_stride, d->bytes)))
    return rc;
  cudaStream_t st = g->stream;
  (void)cudaGetLastError();
  DecodeParams P;
  fill_params(d, P);
  P.n = 1;
  P.slots = d->d_slots;
  P.hyps = d->d_hyps;
  P.hyp_stride = 1;
  P.n_hyps = d->d_nhyps;
  P.errors = d->d_errors;
  P.frames_done = d->d_done;
  P.words = d->d_words;
  P.words_stride = words_stride;
  P.words_used = d->d_wused;
  CK(cudaMemcpyAsync(d->d_slots, &ch, sizeof(int), cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(d->d_wused, 0, sizeof(long long), st));
  P.ctx_words_cap = CTX_SMEM_WORDS;
  P.row_in_smem = 1;
  const size_t smem = CTX_SMEM_WORDS * sizeof(u32);
  cudaError_t le = d->hashed ? (g->fmt16 ? launch_hyp<256, Fmt16<true>, float>(P, which, smem, st)
                                         : launch_hyp<256, Fmt24<true>, float>(P, which, smem, st))
                             : (g->fmt16 ? launch_hyp<256, Fmt16<false>, float>(P, which, smem, st)
                                         : launch_hyp<256, Fmt24<false>, float>(P, which, smem, st));
  if (le != cudaSuccess) return fail(AB_ERR_CUDA, "hypothesis launch: %s", cudaGetErrorString(le));
  int err = 0, nh = 0;
  long long nw = 0;
  DevHyp h;
  CK(cudaMemcpyAsync(&err, d->d_errors, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&nh, d->d_nhyps, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&nw, d->d_wused, sizeof(long long), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&h, d->d_hyps, sizeof(DevHyp), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (err == AB_ERR_DEAD) return fail(AB_ERR_DEAD, "decode failure, no active tokens");
  if (err == AB_ERR_STATUS) return fail(AB_ERR_STATUS, "cannot finalize in this status");
  if (err) return fail(err, "device error %d", err);
  if (nw > words_cap) return fail(AB_ERR_CAPACITY, "words buffer too small");
  if (nw) CK(cudaMemcpy(words, d->d_words, nw * sizeof(int), cudaMemcpyDeviceToHost));
  hyp->cost = h.cost;
  hyp->frame = h.frame;
  hyp->kind = h.kind;
  hyp->fallback = h.fallback;
  hyp->hits = h.hits;
  hyp->shared = h.shared;
  hyp->n_words = h.n_words;
  hyp->pad_ = 0;
  hyp->words_off = 0;
  return AB_OK;
}

extern "C" int ab_partial(ab_decoder *d, int32_t ch, ab_hyp *hyp, int32_t *words,
                          int32_t words_cap) {
  return one_hyp(d, ch, AB_PARTIAL, hyp, words, words_cap);
}

extern "C" int ab_finalize(ab_decoder *d, int32_t ch, ab_hyp *hyp, int32_t *words,
                           int32_t words_cap) {
  return one_hyp(d, ch, AB_FINAL, hyp, words, words_cap);
}

struct ab_fst {
  ab::HostFst F;
};

extern "C" int ab_fst_parse(const char *text, int64_t len, int64_t num_states_hint, ab_fst **out) {
  if (!out || (!text && len)) return fail(AB_ERR_INVALID, "null argument");
  *out = nullptr;
  ab_fst *f = new ab_fst();
  std::string err;
  const int rc = ab::parse_text_fst(text ? text : "", (size_t)std::max<int64_t>(len, 0), num_states_hint, f->F, err);
  if (rc) {
    delete f;
    return fail(rc == 1 ? AB_ERR_PARSE : AB_ERR_STRUCTURE, "%s", err.c_str());
  }
  *out = f;
  return AB_OK;
}

extern "C" int ab_fst_load(const char *path, int64_t num_states_hint, int32_t use_cache, const char *cache_path,
                           int32_t *cache_hit, ab_fst **out) {
  if (!path || !out) return fail(AB_ERR_INVALID, "null argument");
  *out = nullptr;
  if (cache_hit) *cache_hit = 0;
  struct stat st;
  if (stat(path, &st) != 0) return fail(AB_ERR_INVALID, "cannot stat %s", path);
  const int64_t mtime = (int64_t)st.st_mtim.tv_sec * 1000000000ll + st.st_mtim.tv_nsec;
  ab_fst *f = new ab_fst();
  if (use_cache && cache_path && num_states_hint < 0 && ab::load_cache(cache_path, f->F, (int64_t)st.st_size, mtime)) {
    if (cache_hit) *cache_hit = 1;
    *out = f;
    return AB_OK;
  }
  FILE *fp = fopen(path, "rb");
  if (!fp) {
    delete f;
    return fail(AB_ERR_INVALID, "cannot open %s", path);
  }
  std::vector<char> buf((size_t)st.st_size);
  const size_t got = buf.empty() ? 0 : fread(buf.data(), 1, buf.size(), fp);
  fclose(fp);
  if (got != buf.size()) {
    delete f;
    return fail(AB_ERR_INVALID, "short read of %s", path);
  }
  std::string err;
  const int rc = ab::parse_text_fst(buf.data(), buf.size(), num_states_hint, f->F, err);
  if (rc) {
    delete f;
    return fail(rc == 1 ? AB_ERR_PARSE : AB_ERR_STRUCTURE, "%s", err.c_str());
  }
  if (use_cache && cache_path && num_states_hint < 0) ab::save_cache(cache_path, f->F, (int64_t)st.st_size, mtime);
  *out = f;
  return AB_OK;
}

extern "C" int ab_fst_info(const ab_fst *f, int32_t *start, int64_t *num_states, int64_t *num_arcs,
                           int32_t *num_finals, char *fingerprint65) {
  if (!f) return fail(AB_ERR_INVALID, "null fst");
  if (start) *start = f->F.start;
  if (num_states) *num_states = f->F.num_states;
  if (num_arcs) *num_arcs = (int64_t)f->F.il.size();
  if (num_finals) *num_finals = (int32_t)f->F.fstate.size();
  if (fingerprint65) {
    memcpy(fingerprint65, f->F.fingerprint.data(), 64);
    fingerprint65[64] = 0;
  }
  return AB_OK;
}

extern "C" int ab_fst_arrays(const ab_fst *f, int64_t *row_offsets, int32_t *ilabels, int32_t *olabels,
                             int32_t *next_states, double *weights, int32_t *final_states, double *final_costs) {
  if (!f) return fail(AB_ERR_INVALID, "null fst");
  const ab::HostFst &F = f->F;
  if (row_offsets) std::copy(F.ro.begin(), F.ro.end(), row_offsets);
  if (ilabels) std::copy(F.il.begin(), F.il.end(), ilabels);
  if (olabels) std::copy(F.ol.begin(), F.ol.end(), olabels);
  if (next_states) std::copy(F.ns.begin(), F.ns.end(), next_states);
  if (weights) std::copy(F.w.begin(), F.w.end(), weights);
  if (final_states) std::copy(F.fstate.begin(), F.fstate.end(), final_states);
  if (final_costs) std::copy(F.fcost.begin(), F.fcost.end(), final_costs);
  return AB_OK;
}

extern "C" void ab_fst_destroy(ab_fst *f) { delete f; }

extern "C" int ab_graph_create_from_fst(int32_t device, const ab_fst *f, ab_graph **out) {
  if (!f || !out) return fail(AB_ERR_INVALID, "null argument");
  const ab::HostFst &F = f->F;
  if (F.num_states > INT32_MAX) return fail(AB_ERR_INVALID, "too many states");
  return ab_graph_create(device, F.start, (int32_t)F.num_states, (int64_t)F.il.size(), F.ro.data(), F.il.data(),
                         F.ol.data(), F.ns.data(), F.w.data(), (int32_t)F.fstate.size(), F.fstate.data(),
                         F.fcost.data(), out);
}

struct ab_scores {
  ab::HostScores S;
};

extern "C" int ab_scores_parse(const char *text, int64_t len, ab_scores **out) {
  if (!out || (!text && len)) return fail(AB_ERR_INVALID, "null argument");
  *out = nullptr;
  ab_scores *s = new ab_scores();
  std::string err;
  const int rc = ab::parse_score_text(text ? text : "", (size_t)std::max<int64_t>(len, 0), s->S, err);
  if (rc) {
    delete s;
    return fail(rc == 1 ? AB_ERR_SCORE_FORMAT : AB_ERR_INVALID, "%s", err.c_str());
  }
  *out = s;
  return AB_OK;
}

extern "C" int ab_scores_info(const ab_scores *s, int64_t *num_frames, int64_t *num_ilabels,
                              double *frame_duration) {
  if (!s) return fail(AB_ERR_INVALID, "null scores");
  if (num_frames) *num_frames = s->S.T;
  if (num_ilabels) *num_ilabels = s->S.L;
  if (frame_duration) *frame_duration = s->S.dur;
  return AB_OK;
}

extern "C" int ab_scores_copy(const ab_scores *s, double *costs) {
  if (!s || (!costs && !s->S.costs.empty())) return fail(AB_ERR_INVALID, "null argument");
  std::copy(s->S.costs.begin(), s->S.costs.end(), costs);
  return AB_OK;
}

extern "C" void ab_scores_destroy(ab_scores *s) { delete s; }

extern "C" int ab_compile_context(int32_t num_states, int64_t num_arcs, const int64_t *row_offsets,
                                  const int32_t *olabels, const int32_t *next_states,
                                  int32_t n_entities, const int64_t *ent_offsets,
                                  const int32_t *labels, int32_t max_epsilon_depth,
                                  int32_t num_threads, int64_t *out_arcs, int64_t out_cap,
                                  int64_t *n_out, int32_t *ent_status) {
  if (num_states < 1 || num_arcs < 0 || !row_offsets || (num_arcs && (!olabels || !next_states)))
    return fail(AB_ERR_INVALID, "invalid graph arrays");
  if (n_entities < 0 || (n_entities && (!ent_offsets || !ent_status)) || !n_out)
    return fail(AB_ERR_INVALID, "invalid entity arrays");
  if (max_epsilon_depth < 0) return fail(AB_ERR_INVALID, "max_epsilon_depth must be >= 0");
  if (row_offsets[0] != 0 || row_offsets[num_states] != num_arcs)
    return fail(AB_ERR_INVALID, "row_offsets must start at 0 and end at num_arcs");
  for (int64_t a = 0; a < num_arcs; ++a)
    if (olabels[a] < 0 || next_states[a] < 0 || next_states[a] >= num_states)
      return fail(AB_ERR_INVALID, "arc %lld: label or next state out of range", (long long)a);
  for (int32_t e = 0; e < n_entities; ++e)
    if (ent_offsets[e + 1] < ent_offsets[e]) return fail(AB_ERR_INVALID, "entity offsets decrease");
  ab::CompileGraph G{num_states, num_arcs, row_offsets, olabels, next_states};
  G.index();
  int32_t threads = num_threads > 0 ? num_threads : (int32_t)std::max(1u, std::thread::hardware_concurrency());
  const std::vector<int64_t> all = ab::compile_entities(G, n_entities, ent_offsets, labels,
                                                        max_epsilon_depth, threads, ent_status);
  *n_out = (int64_t)all.size();
  if (out_arcs)
    std::copy(all.begin(), all.begin() + std::min<int64_t>((int64_t)all.size(), std::max<int64_t>(out_cap, 0)),
              out_arcs);
  return AB_OK;
}

extern "C" int ab_align(const int32_t *ref, int64_t nr, const int32_t *hyp, int64_t nh, int8_t *kind,
                        int32_t *ref_pos, int32_t *hyp_pos, int64_t cap, int64_t *n_ops) {
  if (nr < 0 || nh < 0 || (nr && !ref) || (nh && !hyp) || !n_ops) return fail(AB_ERR_INVALID, "invalid arguments");
  if (nr >= INT32_MAX || nh >= INT32_MAX) return fail(AB_ERR_INVALID, "sequence too long");
  std::vector<uint32_t> D;
  std::vector<int8_t> k;
  std::vector<int32_t> rp, hp;
  ab::edit_table(ref, nr, hyp, nh, D);
  ab::backtrace(ref, nr, hyp, nh, D, k, rp, hp);
  *n_ops = (int64_t)k.size();
  const size_t m = (size_t)std::min<int64_t>((int64_t)k.size(), std::max<int64_t>(cap, 0));
  if (m && (!kind || !ref_pos || !hyp_pos)) return fail(AB_ERR_INVALID, "null output");
  std::copy(k.begin(), k.begin() + m, kind);
  std::copy(rp.begin(), rp.begin() + m, ref_pos);
  std::copy(hp.begin(), hp.begin() + m, hyp_pos);
  return AB_OK;
}

extern "C" int ab_edit_distances(int64_t n, const int64_t *ref_off, const int32_t *ref, const int64_t *hyp_off,
                                 const int32_t *hyp, int32_t num_threads, int64_t *dist) {
  if (n < 0 || (n && (!ref_off || !hyp_off || !dist))) return fail(AB_ERR_INVALID, "invalid arguments");
  for (int64_t p = 0; p < n; ++p)
    if (ref_off[p + 1] < ref_off[p] || hyp_off[p + 1] < hyp_off[p]) return fail(AB_ERR_INVALID, "offsets decrease");
  if (n && ((ref_off[n] > ref_off[0] && !ref) || (hyp_off[n] > hyp_off[0] && !hyp)))
    return fail(AB_ERR_INVALID, "null word array");
  const int32_t threads = num_threads > 0 ? num_threads : (int32_t)std::max(1u, std::thread::hardware_concurrency());
  ab::edit_distances(n, ref_off, ref, hyp_off, hyp, threads, dist);
  return AB_OK;
}

extern "C" int ab_scores_generate(int32_t device, const uint64_t *streams, int32_t n_streams,
                                  int64_t values_per_stream, double low, double high, double offset,
                                  int32_t dtype, void *out, void *stream) {
  if (n_streams < 0 || values_per_stream < 0 || (n_streams && (!streams || !out)))
    return fail(AB_ERR_INVALID, "invalid arguments");
  if (dtype != AB_F32 && dtype != AB_F64) return fail(AB_ERR_INVALID, "dtype must be AB_F32 or AB_F64");
  if (!n_streams || !values_per_stream) return AB_OK;
  CK(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long *d_streams = nullptr;
  CK(cudaMalloc(&d_streams, (size_t)n_streams * 4 * sizeof(unsigned long long)));
  cudaError_t e = cudaMemcpyAsync(d_streams, streams, (size_t)n_streams * 4 * sizeof(unsigned long long),
                                  cudaMemcpyHostToDevice, st);
  const long long chunks = (values_per_stream + ab::GEN_CHUNK - 1) / ab::GEN_CHUNK;
  const long long threads = chunks * n_streams;
  const unsigned blocks = (unsigned)((threads + 255) / 256);
  if (e == cudaSuccess) {
    if (dtype == AB_F32)
      ab::uniform_kernel<float><<<blocks, 256, 0, st>>>(d_streams, n_streams, values_per_stream, low, high - low,
                                                        offset, (float *)out);
    else
      ab::uniform_kernel<double><<<blocks, 256, 0, st>>>(d_streams, n_streams, values_per_stream, low, high - low,
                                                         offset, (double *)out);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(d_streams);
  if (e != cudaSuccess) return fail(AB_ERR_CUDA, "score generation: %s", cudaGetErrorString(e));
  return AB_OK;
}

extern "C" int ab_last_kernel_ms(ab_decoder *d, float *ms) {
  if (!d) return fail(AB_ERR_INVALID, "null decoder");
  *ms = d->last_ms;
  return AB_OK;
}

extern "C" int ab_last_launch_count(ab_decoder *d, int32_t *launches) {
  if (!d) return fail(AB_ERR_INVALID, "null decoder");
  *launches = d->last_launches;
  return AB_OK;
}
