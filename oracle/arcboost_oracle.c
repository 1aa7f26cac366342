/*
 * arcboost CPU oracle — TEST INFRASTRUCTURE ONLY (see arcboost_oracle.h).
 *
 * Restates /root/reference/pkg/src/arcboost/decoder.py frame by frame.  The
 * reference keeps its token table sorted by state and recombines with
 * np.lexsort; this restatement keeps the same table semantics with a dense
 * state->position map and per-destination running minima, which select the
 * identical winners (minimum (cost, global arc id), decoder.py:213-220) and
 * create emission records in the same order (winners ordered by state).
 */
#include "arcboost_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

struct orc_channel {
  int32_t num_states;
  /* token table (decoder.py:135-138), unordered + pos map */
  int64_t n, cap;
  int32_t *states;
  double *costs;
  int64_t *bp;
  int32_t *last_il;
  int64_t *hits;
  int32_t *pos; /* [num_states] -> index in table or -1 */
  /* lifecycle (decoder.py:119-139) */
  int32_t fresh, status;
  int64_t frame_index, total_frames, utterance_index, trailing_silence, eps_truncations;
  /* EmissionStore (decoder.py:72-107) */
  int64_t rec_n, rec_cap;
  int32_t *rec_ol;
  int64_t *rec_prev;
  /* candidate scratch */
  int64_t c_n, c_cap;
  double *c_cost;
  int64_t *c_arc;
  int32_t *c_src;
  int32_t *c_dst;
  int32_t *best; /* [num_states] -> candidate index or -1 */
  int64_t *radix_cnt; /* [1 << 16] */
  int64_t w_n, w_cap;
  uint32_t *win, *win_tmp; /* touched destination states */
  /* frontier (decoder.py:254-257) */
  int64_t f_n, f_cap;
  int32_t *f_states;
  double *f_costs;
  int64_t *f_bp;
  int32_t *f_last;
  int64_t *f_hits;
  int64_t *f2_bp;
  /* counters of the last advance */
  int64_t cnt_tok, cnt_emit, cnt_eps;
};

#define GROW(ptr, cap_needed, cap_var, type)                                   \
  do {                                                                         \
    if ((cap_needed) > (cap_var)) {                                            \
      int64_t nc = (cap_var) ? (cap_var) : 64;                                 \
      while (nc < (cap_needed)) nc *= 2;                                       \
      void *np_ = realloc((ptr), (size_t)nc * sizeof(type));                   \
      if (!np_) return ORC_ERR_ALLOC;                                          \
      (ptr) = (type *)np_;                                                     \
      (cap_var) = nc;                                                          \
    }                                                                          \
  } while (0)

static int ensure_table(orc_channel *ch, int64_t need) {
  if (need <= ch->cap) return ORC_OK;
  int64_t nc = ch->cap ? ch->cap : 64;
  while (nc < need) nc *= 2;
  void *a = realloc(ch->states, nc * sizeof(int32_t));
  if (!a) return ORC_ERR_ALLOC;
  ch->states = a;
  a = realloc(ch->costs, nc * sizeof(double));
  if (!a) return ORC_ERR_ALLOC;
  ch->costs = a;
  a = realloc(ch->bp, nc * sizeof(int64_t));
  if (!a) return ORC_ERR_ALLOC;
  ch->bp = a;
  a = realloc(ch->last_il, nc * sizeof(int32_t));
  if (!a) return ORC_ERR_ALLOC;
  ch->last_il = a;
  a = realloc(ch->hits, nc * sizeof(int64_t));
  if (!a) return ORC_ERR_ALLOC;
  ch->hits = a;
  ch->cap = nc;
  return ORC_OK;
}

static int ensure_cands(orc_channel *ch, int64_t need) {
  if (need <= ch->c_cap) return ORC_OK;
  int64_t nc = ch->c_cap ? ch->c_cap : 256;
  while (nc < need) nc *= 2;
  void *a = realloc(ch->c_cost, nc * sizeof(double));
  if (!a) return ORC_ERR_ALLOC;
  ch->c_cost = a;
  a = realloc(ch->c_arc, nc * sizeof(int64_t));
  if (!a) return ORC_ERR_ALLOC;
  ch->c_arc = a;
  a = realloc(ch->c_src, nc * sizeof(int32_t));
  if (!a) return ORC_ERR_ALLOC;
  ch->c_src = a;
  a = realloc(ch->c_dst, nc * sizeof(int32_t));
  if (!a) return ORC_ERR_ALLOC;
  ch->c_dst = a;
  ch->c_cap = nc;
  return ORC_OK;
}

static int ensure_frontier(orc_channel *ch, int64_t need) {
  if (need <= ch->f_cap) return ORC_OK;
  int64_t nc = ch->f_cap ? ch->f_cap : 64;
  while (nc < need) nc *= 2;
  void *a = realloc(ch->f_states, nc * sizeof(int32_t));
  if (!a) return ORC_ERR_ALLOC;
  ch->f_states = a;
  a = realloc(ch->f_costs, nc * sizeof(double));
  if (!a) return ORC_ERR_ALLOC;
  ch->f_costs = a;
  a = realloc(ch->f_bp, nc * sizeof(int64_t));
  if (!a) return ORC_ERR_ALLOC;
  ch->f_bp = a;
  a = realloc(ch->f_last, nc * sizeof(int32_t));
  if (!a) return ORC_ERR_ALLOC;
  ch->f_last = a;
  a = realloc(ch->f_hits, nc * sizeof(int64_t));
  if (!a) return ORC_ERR_ALLOC;
  ch->f_hits = a;
  a = realloc(ch->f2_bp, nc * sizeof(int64_t));
  if (!a) return ORC_ERR_ALLOC;
  ch->f2_bp = a;
  ch->f_cap = nc;
  return ORC_OK;
}

orc_channel *orc_channel_new(const orc_graph *g) {
  orc_channel *ch = (orc_channel *)calloc(1, sizeof(orc_channel));
  if (!ch) return NULL;
  ch->num_states = g->num_states;
  int64_t ns = g->num_states > 0 ? g->num_states : 1;
  ch->pos = (int32_t *)malloc(ns * sizeof(int32_t));
  ch->best = (int32_t *)malloc(ns * sizeof(int32_t));
  ch->radix_cnt = (int64_t *)malloc(sizeof(int64_t) << 16);
  if (!ch->pos || !ch->best || !ch->radix_cnt) {
    orc_channel_free(ch);
    return NULL;
  }
  for (int64_t i = 0; i < ns; ++i) ch->pos[i] = -1, ch->best[i] = -1;
  ch->fresh = 1;
  ch->status = ORC_IDLE;
  return ch;
}

void orc_channel_free(orc_channel *ch) {
  if (!ch) return;
  free(ch->states); free(ch->costs); free(ch->bp); free(ch->last_il); free(ch->hits);
  free(ch->pos); free(ch->rec_ol); free(ch->rec_prev);
  free(ch->c_cost); free(ch->c_arc); free(ch->c_src); free(ch->c_dst); free(ch->best);
  free(ch->win); free(ch->win_tmp);
  free(ch->f_states); free(ch->f_costs); free(ch->f_bp); free(ch->f_last); free(ch->f_hits);
  free(ch->f2_bp); free(ch->radix_cnt);
  free(ch);
}

void orc_channel_get_info(const orc_channel *ch, orc_channel_info *o) {
  o->status = ch->status;
  o->fresh = ch->fresh;
  o->frame_index = ch->frame_index;
  o->total_frames = ch->total_frames;
  o->utterance_index = ch->utterance_index;
  o->trailing_silence = ch->trailing_silence;
  o->eps_truncations = ch->eps_truncations;
  o->num_active = ch->n;
  o->store_len = ch->rec_n;
  o->tok_expansions = ch->cnt_tok;
  o->emit_arcs = ch->cnt_emit;
  o->eps_arcs = ch->cnt_eps;
}

void orc_channel_set_status(orc_channel *ch, int32_t s) { ch->status = s; }
void orc_channel_set_trailing_silence(orc_channel *ch, int64_t v) { ch->trailing_silence = v; }

/* EmissionStore.append (decoder.py:85-90); frame ids are not kept (unused by backtrace). */
static int64_t rec_append(orc_channel *ch, int32_t ol, int64_t prev) {
  if (ch->rec_n == ch->rec_cap) {
    int64_t nc = ch->rec_cap ? 2 * ch->rec_cap : 1024;
    void *a = realloc(ch->rec_ol, nc * sizeof(int32_t));
    if (!a) return -2;
    ch->rec_ol = a;
    a = realloc(ch->rec_prev, nc * sizeof(int64_t));
    if (!a) return -2;
    ch->rec_prev = a;
    ch->rec_cap = nc;
  }
  ch->rec_ol[ch->rec_n] = ol;
  ch->rec_prev[ch->rec_n] = prev;
  return ch->rec_n++;
}

/* BiasingContext.boosted_mask / sorted_contains (biasing.py:108-117, 140-163). */
static inline int is_boosted(const orc_context *ctx, int64_t g) {
  int64_t lo = 0, hi = ctx->k;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    int64_t v = ctx->arc_indices[mid];
    if (v == g) return 1;
    if (v < g) lo = mid + 1;
    else hi = mid;
  }
  return 0;
}

/* _effective_weights (decoder.py:234-240), see the signed-zero note in the header. */
static inline double eff_weight(const orc_graph *g, const orc_context *ctx, int64_t arc,
                                int *boosted) {
  double w = g->weights[arc];
  *boosted = 0;
  if (ctx && ctx->k > 0 && is_boosted(ctx, arc)) {
    *boosted = 1;
    w = w + ctx->discount;
  }
  return w;
}

/* Candidate bookkeeping for _recombine (decoder.py:213-220): per destination the
 * winner minimises (cost, global arc id). */
static inline void offer(orc_channel *ch, int32_t d, double c, int64_t arc, int32_t src) {
  int64_t k = ch->c_n++;
  ch->c_cost[k] = c;
  ch->c_arc[k] = arc;
  ch->c_src[k] = src;
  ch->c_dst[k] = d;
  int32_t b = ch->best[d];
  if (b < 0) {
    ch->best[d] = (int32_t)k;
    ch->win[ch->w_n++] = (uint32_t)d;
  } else if (c < ch->c_cost[b] || (c == ch->c_cost[b] && arc < ch->c_arc[b])) {
    ch->best[d] = (int32_t)k;
  }
}

/* Winners are visited in state order, as np.lexsort(..., states) leaves them. */
static void sort_winners(orc_channel *ch) {
  int64_t n = ch->w_n;
  if (n < 64) {
    for (int64_t i = 1; i < n; ++i) {
      uint32_t v = ch->win[i];
      int64_t j = i - 1;
      while (j >= 0 && ch->win[j] > v) {
        ch->win[j + 1] = ch->win[j];
        --j;
      }
      ch->win[j + 1] = v;
    }
    return;
  }
  static const int B = 16;
  uint32_t *a = ch->win, *t = ch->win_tmp;
  int64_t *cnt = ch->radix_cnt;
  for (int pass = 0; pass < 2; ++pass) {
    memset(cnt, 0, sizeof(int64_t) << 16);
    int sh = pass * B;
    for (int64_t i = 0; i < n; ++i) cnt[(a[i] >> sh) & 0xFFFF]++;
    int64_t s = 0;
    for (int i = 0; i < (1 << 16); ++i) {
      int64_t c = cnt[i];
      cnt[i] = s;
      s += c;
    }
    for (int64_t i = 0; i < n; ++i) t[cnt[(a[i] >> sh) & 0xFFFF]++] = a[i];
    uint32_t *x = a;
    a = t;
    t = x;
  }
  /* two passes: result back in ch->win */
}

static int ensure_win(orc_channel *ch, int64_t need) {
  if (need <= ch->w_cap) return ORC_OK;
  int64_t nc = ch->w_cap ? ch->w_cap : 256;
  while (nc < need) nc *= 2;
  void *a = realloc(ch->win, nc * sizeof(uint32_t));
  if (!a) return ORC_ERR_ALLOC;
  ch->win = a;
  a = realloc(ch->win_tmp, nc * sizeof(uint32_t));
  if (!a) return ORC_ERR_ALLOC;
  ch->win_tmp = a;
  ch->w_cap = nc;
  return ORC_OK;
}

static void clear_table(orc_channel *ch) {
  for (int64_t i = 0; i < ch->n; ++i) ch->pos[ch->states[i]] = -1;
  ch->n = 0;
}

/* _materialize_start (decoder.py:243-247). */
static int materialize_start(orc_channel *ch, const orc_graph *g) {
  clear_table(ch);
  int rc = ensure_table(ch, 1);
  if (rc) return rc;
  ch->states[0] = g->start;
  ch->costs[0] = 0.0;
  ch->bp[0] = -1;
  ch->last_il[0] = 0;
  ch->hits[0] = 0;
  ch->pos[g->start] = 0;
  ch->n = 1;
  return ORC_OK;
}

/* _epsilon_rounds (decoder.py:250-316): synchronous rounds over epsilon-input arcs;
 * a round winner is applied iff its state is new or it is strictly cheaper. */
static int epsilon_rounds(orc_channel *ch, const orc_graph *g, const orc_context *ctx,
                          const orc_config *cfg) {
  int rc = ensure_frontier(ch, ch->n);
  if (rc) return rc;
  int64_t nf = ch->n;
  memcpy(ch->f_states, ch->states, nf * sizeof(int32_t));
  memcpy(ch->f_costs, ch->costs, nf * sizeof(double));
  memcpy(ch->f_bp, ch->bp, nf * sizeof(int64_t));
  memcpy(ch->f_last, ch->last_il, nf * sizeof(int32_t));
  memcpy(ch->f_hits, ch->hits, nf * sizeof(int64_t));
  int rounds = 0;
  for (;;) {
    if (!(nf > 0 && rounds < cfg->max_eps)) {
      if (nf > 0) ch->eps_truncations += 1; /* while-else, decoder.py:314-316 */
      break;
    }
    rounds++;
    /* _gather_arcs + il == 0 filter (decoder.py:261-267) */
    int64_t need = 0;
    for (int64_t i = 0; i < nf; ++i) {
      int32_t s = ch->f_states[i];
      need += g->row_offsets[s + 1] - g->row_offsets[s];
    }
    ch->cnt_tok += nf;
    if ((rc = ensure_cands(ch, need)) || (rc = ensure_win(ch, need))) return rc;
    ch->c_n = 0;
    ch->w_n = 0;
    for (int64_t i = 0; i < nf; ++i) {
      int32_t s = ch->f_states[i];
      for (int64_t a = g->row_offsets[s]; a < g->row_offsets[s + 1]; ++a) {
        if (g->ilabels[a] != 0) continue;
        int bst;
        double c = ch->f_costs[i] + eff_weight(g, ctx, a, &bst); /* decoder.py:268 */
        ch->cnt_eps++;
        offer(ch, g->next_states[a], c, a, (int32_t)i);
      }
    }
    if (ch->c_n == 0) break; /* decoder.py:263-265 */
    sort_winners(ch);
    /* strict-improvement apply (decoder.py:277-287) */
    int64_t n_app = 0;
    int64_t nw = ch->w_n;
    /* reuse win_tmp as the applied list of winner-candidate ids */
    for (int64_t w = 0; w < nw; ++w) {
      int32_t d = (int32_t)ch->win[w];
      int32_t k = ch->best[d];
      int32_t p = ch->pos[d];
      if (p < 0 || ch->c_cost[k] < ch->costs[p]) ch->win_tmp[n_app++] = (uint32_t)k;
    }
    for (int64_t w = 0; w < nw; ++w) ch->best[ch->win[w]] = -1;
    if (n_app == 0) break;
    /* records for applied winners with olabel != 0, in state order (decoder.py:289-295) */
    if ((rc = ensure_table(ch, ch->n + n_app))) return rc;
    for (int64_t j = 0; j < n_app; ++j) {
      int32_t k = (int32_t)ch->win_tmp[j];
      int64_t arc = ch->c_arc[k];
      int32_t src = ch->c_src[k];
      int32_t ol = g->olabels[arc];
      int64_t nbp = ch->f_bp[src];
      if (ol != 0) {
        nbp = rec_append(ch, ol, nbp);
        if (nbp == -2) return ORC_ERR_ALLOC;
      }
      ch->f2_bp[j] = nbp;
    }
    /* apply (decoder.py:297-308); then the applied winners form the next frontier */
    for (int64_t j = 0; j < n_app; ++j) {
      int32_t k = (int32_t)ch->win_tmp[j];
      int64_t arc = ch->c_arc[k];
      int32_t src = ch->c_src[k];
      int32_t d = ch->c_dst[k];
      int bst = 0;
      if (ctx && ctx->k > 0) bst = is_boosted(ctx, arc);
      int32_t p = ch->pos[d];
      if (p < 0) {
        p = (int32_t)ch->n++;
        ch->states[p] = d;
        ch->pos[d] = p;
      }
      ch->costs[p] = ch->c_cost[k];
      ch->bp[p] = ch->f2_bp[j];
      ch->last_il[p] = ch->f_last[src];
      ch->hits[p] = ch->f_hits[src] + bst;
    }
    /* new frontier; gather sources first (in-place hazard) */
    if ((rc = ensure_frontier(ch, n_app))) return rc;
    {
      /* stage into temporaries in candidate arrays' spare room is unsafe; use per-j copies */
      int32_t *ns = (int32_t *)malloc(n_app * sizeof(int32_t));
      double *nc = (double *)malloc(n_app * sizeof(double));
      int32_t *nl = (int32_t *)malloc(n_app * sizeof(int32_t));
      int64_t *nh = (int64_t *)malloc(n_app * sizeof(int64_t));
      if (!ns || !nc || !nl || !nh) {
        free(ns); free(nc); free(nl); free(nh);
        return ORC_ERR_ALLOC;
      }
      for (int64_t j = 0; j < n_app; ++j) {
        int32_t k = (int32_t)ch->win_tmp[j];
        int32_t src = ch->c_src[k];
        int bst = 0;
        if (ctx && ctx->k > 0) bst = is_boosted(ctx, ch->c_arc[k]);
        ns[j] = ch->c_dst[k];
        nc[j] = ch->c_cost[k];
        nl[j] = ch->f_last[src];
        nh[j] = ch->f_hits[src] + bst;
      }
      memcpy(ch->f_states, ns, n_app * sizeof(int32_t));
      memcpy(ch->f_costs, nc, n_app * sizeof(double));
      memcpy(ch->f_last, nl, n_app * sizeof(int32_t));
      memcpy(ch->f_hits, nh, n_app * sizeof(int64_t));
      memcpy(ch->f_bp, ch->f2_bp, n_app * sizeof(int64_t));
      free(ns); free(nc); free(nl); free(nh);
    }
    nf = n_app;
  }
  return ORC_OK;
}

/* (cost, state) order used by _prune, _best_token_pos and finalize (decoder.py:327,338,447). */
static int cmp_cost_state_ctx_less(double ca, int32_t sa, double cb, int32_t sb) {
  return ca < cb || (ca == cb && sa < sb);
}

typedef struct {
  double cost;
  int32_t state;
  int32_t idx;
} cs_t;

static int cmp_cs(const void *a, const void *b) {
  const cs_t *x = (const cs_t *)a, *y = (const cs_t *)b;
  if (x->cost < y->cost) return -1;
  if (x->cost > y->cost) return 1;
  return (x->state > y->state) - (x->state < y->state);
}
static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

/* _prune (decoder.py:319-334): beam around the best cost, then max_active by (cost, state). */
static int prune(orc_channel *ch, const orc_config *cfg) {
  if (ch->n == 0) return ORC_OK;
  double best = ch->costs[0];
  for (int64_t i = 1; i < ch->n; ++i)
    if (ch->costs[i] < best) best = ch->costs[i];
  double thr = best + cfg->beam;
  int64_t nk = 0;
  for (int64_t i = 0; i < ch->n; ++i) nk += ch->costs[i] <= thr;
  int32_t *chosen = (int32_t *)malloc((nk ? nk : 1) * sizeof(int32_t));
  if (!chosen) return ORC_ERR_ALLOC;
  int64_t m = 0;
  if (nk > cfg->max_active) {
    cs_t *v = (cs_t *)malloc(nk * sizeof(cs_t));
    if (!v) {
      free(chosen);
      return ORC_ERR_ALLOC;
    }
    int64_t q = 0;
    for (int64_t i = 0; i < ch->n; ++i)
      if (ch->costs[i] <= thr) v[q].cost = ch->costs[i], v[q].state = ch->states[i], v[q].idx = (int32_t)i, q++;
    qsort(v, nk, sizeof(cs_t), cmp_cs);
    for (int64_t i = 0; i < cfg->max_active; ++i) chosen[m++] = v[i].idx;
    free(v);
  } else {
    for (int64_t i = 0; i < ch->n; ++i)
      if (ch->costs[i] <= thr) chosen[m++] = (int32_t)i;
  }
  /* keep the table ordered by state like the reference (np.sort(idx), states sorted) */
  int32_t *st = (int32_t *)malloc((m ? m : 1) * sizeof(int32_t));
  if (!st) {
    free(chosen);
    return ORC_ERR_ALLOC;
  }
  for (int64_t i = 0; i < m; ++i) st[i] = ch->states[chosen[i]];
  qsort(st, m, sizeof(int32_t), cmp_i32);
  /* gather survivors by state through the pos map */
  double *nc = (double *)malloc((m ? m : 1) * sizeof(double));
  int64_t *nb = (int64_t *)malloc((m ? m : 1) * sizeof(int64_t));
  int32_t *nl = (int32_t *)malloc((m ? m : 1) * sizeof(int32_t));
  int64_t *nh = (int64_t *)malloc((m ? m : 1) * sizeof(int64_t));
  if (!nc || !nb || !nl || !nh) {
    free(chosen); free(st); free(nc); free(nb); free(nl); free(nh);
    return ORC_ERR_ALLOC;
  }
  for (int64_t i = 0; i < m; ++i) {
    int32_t p = ch->pos[st[i]];
    nc[i] = ch->costs[p];
    nb[i] = ch->bp[p];
    nl[i] = ch->last_il[p];
    nh[i] = ch->hits[p];
  }
  clear_table(ch);
  for (int64_t i = 0; i < m; ++i) {
    ch->states[i] = st[i];
    ch->costs[i] = nc[i];
    ch->bp[i] = nb[i];
    ch->last_il[i] = nl[i];
    ch->hits[i] = nh[i];
    ch->pos[st[i]] = (int32_t)i;
  }
  ch->n = m;
  free(chosen); free(st); free(nc); free(nb); free(nl); free(nh);
  return ORC_OK;
}

/* _best_token_pos (decoder.py:337-338). */
static int64_t best_pos(const orc_channel *ch) {
  int64_t b = 0;
  for (int64_t i = 1; i < ch->n; ++i)
    if (cmp_cost_state_ctx_less(ch->costs[i], ch->states[i], ch->costs[b], ch->states[b])) b = i;
  return b;
}

/* advance_frame (decoder.py:341-411). */
int orc_advance(orc_channel *ch, const orc_graph *g, const orc_context *ctx,
                const orc_config *cfg, const double *row, int64_t width) {
  if (ch->status != ORC_IDLE && ch->status != ORC_DECODING) return ORC_ERR_STATUS;
  if (width != g->num_emitting_labels) return ORC_ERR_WIDTH;
  int rc;
  ch->cnt_tok = ch->cnt_emit = ch->cnt_eps = 0;
  if (ch->fresh) {
    if ((rc = materialize_start(ch, g))) return rc;
    if ((rc = epsilon_rounds(ch, g, ctx, cfg))) return rc; /* utterance-start closure, no prune */
    ch->fresh = 0;
  }
  ch->status = ORC_DECODING;

  /* emitting pass (decoder.py:367-398) */
  int64_t need = 0;
  for (int64_t i = 0; i < ch->n; ++i) {
    int32_t s = ch->states[i];
    need += g->row_offsets[s + 1] - g->row_offsets[s];
  }
  ch->cnt_tok += ch->n;
  if ((rc = ensure_cands(ch, need)) || (rc = ensure_win(ch, need))) return rc;
  ch->c_n = 0;
  ch->w_n = 0;
  for (int64_t i = 0; i < ch->n; ++i) {
    int32_t s = ch->states[i];
    for (int64_t a = g->row_offsets[s]; a < g->row_offsets[s + 1]; ++a) {
      int32_t il = g->ilabels[a];
      if (il == 0) continue;
      int bst;
      double c = (ch->costs[i] + eff_weight(g, ctx, a, &bst)) + row[il - 1]; /* decoder.py:378 */
      ch->cnt_emit++;
      offer(ch, g->next_states[a], c, a, (int32_t)i);
    }
  }
  sort_winners(ch);
  int64_t nw = ch->w_n;
  /* the new table is exactly the winners (tokens without emitting arcs die) */
  int32_t *ns = (int32_t *)malloc((nw ? nw : 1) * sizeof(int32_t));
  double *nc = (double *)malloc((nw ? nw : 1) * sizeof(double));
  int64_t *nb = (int64_t *)malloc((nw ? nw : 1) * sizeof(int64_t));
  int32_t *nl = (int32_t *)malloc((nw ? nw : 1) * sizeof(int32_t));
  int64_t *nh = (int64_t *)malloc((nw ? nw : 1) * sizeof(int64_t));
  if (!ns || !nc || !nb || !nl || !nh) {
    free(ns); free(nc); free(nb); free(nl); free(nh);
    return ORC_ERR_ALLOC;
  }
  for (int64_t w = 0; w < nw; ++w) {
    int32_t d = (int32_t)ch->win[w];
    int32_t k = ch->best[d];
    int64_t arc = ch->c_arc[k];
    int32_t src = ch->c_src[k];
    int32_t ol = g->olabels[arc];
    int64_t nbp = ch->bp[src];
    if (ol != 0) {
      nbp = rec_append(ch, ol, nbp); /* decoder.py:385-389 */
      if (nbp == -2) {
        free(ns); free(nc); free(nb); free(nl); free(nh);
        return ORC_ERR_ALLOC;
      }
    }
    int bst = 0;
    if (ctx && ctx->k > 0) bst = is_boosted(ctx, arc);
    ns[w] = d;
    nc[w] = ch->c_cost[k];
    nb[w] = nbp;
    nl[w] = g->ilabels[arc];
    nh[w] = ch->hits[src] + bst;
  }
  for (int64_t w = 0; w < nw; ++w) ch->best[ch->win[w]] = -1;
  clear_table(ch);
  if ((rc = ensure_table(ch, nw))) {
    free(ns); free(nc); free(nb); free(nl); free(nh);
    return rc;
  }
  for (int64_t w = 0; w < nw; ++w) {
    ch->states[w] = ns[w];
    ch->costs[w] = nc[w];
    ch->bp[w] = nb[w];
    ch->last_il[w] = nl[w];
    ch->hits[w] = nh[w];
    ch->pos[ns[w]] = (int32_t)w;
  }
  ch->n = nw;
  free(ns); free(nc); free(nb); free(nl); free(nh);

  if (ch->n > 0) {
    if ((rc = epsilon_rounds(ch, g, ctx, cfg))) return rc;
    if ((rc = prune(ch, cfg))) return rc;
    int64_t b = best_pos(ch);
    if (cfg->silence_ilabel > 0 && ch->last_il[b] == cfg->silence_ilabel)
      ch->trailing_silence += 1;
    else
      ch->trailing_silence = 0;
  }
  ch->frame_index += 1;
  ch->total_frames += 1;
  return ORC_OK;
}

int64_t orc_tokens(const orc_channel *ch, int32_t *states, double *costs, int64_t *hits,
                   int64_t cap) {
  int64_t m = ch->n < cap ? ch->n : cap;
  for (int64_t i = 0; i < m; ++i) {
    if (states) states[i] = ch->states[i];
    if (costs) costs[i] = ch->costs[i];
    if (hits) hits[i] = ch->hits[i];
  }
  return ch->n;
}

/* EmissionStore.backtrace (decoder.py:95-102). */
static int backtrace(const orc_channel *ch, int64_t rec, int32_t *words, int64_t cap,
                     int64_t *n_out) {
  int64_t n = 0;
  for (int64_t i = rec; i >= 0; i = ch->rec_prev[i]) n++;
  if (n > cap) return ORC_ERR_CAPACITY;
  int64_t k = n;
  for (int64_t i = rec; i >= 0; i = ch->rec_prev[i]) words[--k] = ch->rec_ol[i];
  *n_out = n;
  return ORC_OK;
}

/* partial_hypothesis (decoder.py:414-423). */
int orc_partial(orc_channel *ch, orc_hyp *hyp, int32_t *words, int64_t words_cap) {
  hyp->kind = ORC_PARTIAL;
  hyp->fallback = 0;
  hyp->frame = ch->total_frames;
  if (ch->fresh) {
    hyp->cost = 0.0;
    hyp->hits = 0;
    hyp->n_words = 0;
    return ORC_OK;
  }
  if (ch->n == 0) return ORC_ERR_DEAD;
  int64_t b = best_pos(ch);
  hyp->cost = ch->costs[b];
  hyp->hits = ch->hits[b];
  return backtrace(ch, ch->bp[b], words, words_cap, &hyp->n_words);
}

/* finalize (decoder.py:426-460). */
int orc_finalize(orc_channel *ch, const orc_graph *g, orc_hyp *hyp, int32_t *words,
                 int64_t words_cap) {
  if (ch->status != ORC_DECODING && ch->status != ORC_ENDPOINTED &&
      !(ch->status == ORC_IDLE && ch->fresh))
    return ORC_ERR_STATUS;
  int rc;
  if (ch->fresh) {
    if ((rc = materialize_start(ch, g))) return rc; /* zero-frame utterance: bare start */
    ch->fresh = 0;
  }
  if (ch->n == 0) return ORC_ERR_DEAD;
  int64_t b = -1;
  double bt = 0.0;
  for (int64_t i = 0; i < ch->n; ++i) {
    int32_t s = ch->states[i];
    if (!g->is_final[s]) continue;
    double t = ch->costs[i] + g->final_costs[s];
    if (b < 0 || cmp_cost_state_ctx_less(t, s, bt, ch->states[b])) b = i, bt = t;
  }
  hyp->kind = ORC_FINAL;
  hyp->frame = ch->total_frames;
  if (b >= 0) {
    hyp->cost = ch->costs[b] + g->final_costs[ch->states[b]];
    hyp->fallback = 0;
  } else {
    b = best_pos(ch);
    hyp->cost = ch->costs[b];
    hyp->fallback = 1;
  }
  hyp->hits = ch->hits[b];
  if ((rc = backtrace(ch, ch->bp[b], words, words_cap, &hyp->n_words))) return rc;
  /* _reset_utterance (decoder.py:151-159) */
  clear_table(ch);
  ch->fresh = 1;
  ch->frame_index = 0;
  ch->trailing_silence = 0;
  ch->rec_n = 0;
  ch->utterance_index += 1;
  ch->status = ORC_IDLE;
  return ORC_OK;
}

/* _decode_one (decoder.py:474-501). */
int orc_decode_stream(orc_channel *ch, const orc_graph *g, const orc_context *ctx,
                      const orc_config *cfg, const double *scores, int64_t T, int64_t width,
                      orc_hyp *hyps, int64_t hyp_cap, int64_t *n_hyps, int32_t *words,
                      int64_t words_cap, int64_t *n_words) {
  *n_hyps = 0;
  *n_words = 0;
  if (ch->status == ORC_FINISHED) ch->status = ORC_IDLE;
  int rc;
  for (int64_t t = 0; t < T; ++t) {
    if ((rc = orc_advance(ch, g, ctx, cfg, scores + t * width, width))) return rc;
    if (ch->frame_index % cfg->partial_every == 0) {
      if (*n_hyps >= hyp_cap) return ORC_ERR_CAPACITY;
      orc_hyp *h = &hyps[*n_hyps];
      if ((rc = orc_partial(ch, h, words + *n_words, words_cap - *n_words))) return rc;
      h->words_off = *n_words;
      *n_words += h->n_words;
      (*n_hyps)++;
    }
    if (ch->trailing_silence >= cfg->endpoint_silence_frames) { /* detect_endpoint 463-464 */
      ch->status = ORC_ENDPOINTED;
      if (*n_hyps >= hyp_cap) return ORC_ERR_CAPACITY;
      orc_hyp *h = &hyps[*n_hyps];
      if ((rc = orc_finalize(ch, g, h, words + *n_words, words_cap - *n_words))) return rc;
      h->words_off = *n_words;
      *n_words += h->n_words;
      (*n_hyps)++;
    }
  }
  if (ch->frame_index > 0 || T == 0) {
    if (*n_hyps >= hyp_cap) return ORC_ERR_CAPACITY;
    orc_hyp *h = &hyps[*n_hyps];
    if ((rc = orc_finalize(ch, g, h, words + *n_words, words_cap - *n_words))) return rc;
    h->words_off = *n_words;
    *n_words += h->n_words;
    (*n_hyps)++;
  }
  ch->status = ORC_FINISHED;
  return ORC_OK;
}
