/*
 * arcboost CPU oracle — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference decoder's per-frame algorithm
 * (/root/reference/pkg/src/arcboost/decoder.py) used as the parity checker
 * for the CUDA path and as the CPU baseline arm of bench.py.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it; the product path (paper_2306_15685_b200) never does.
 *
 * Parity is pinned against the reference itself: tests/golden/make_golden.py
 * imports the reference package in the build container and records its
 * outputs on fixed inputs; tests/test_oracle_golden.py checks this oracle
 * against those fixtures bit-for-bit (costs compared as IEEE doubles).
 *
 * Deliberate extension: every token also carries `hits`, the number of
 * boosted arcs on its path (north-star "boosted-arc hits").  The reference has
 * no such counter; it is carried through exactly the same winner selection as
 * the cost, so it does not influence any reference-visible result.
 *
 * Signed zero: the reference computes w + discount*mask only when some arc of
 * the gathered batch is boosted (decoder.py:234-240), which can turn a -0.0
 * weight into +0.0.  This oracle (like the CUDA path) uses w + discount for
 * boosted arcs and w otherwise; the two differ at most in the sign of a zero
 * cost, which compares equal everywhere in the algorithm.
 */
#ifndef ARCBOOST_ORACLE_H
#define ARCBOOST_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* CsrFst (fst.py:116-162): state-major CSR; global arc index g = row_offsets[s] + j. */
typedef struct orc_graph {
  int32_t start;
  int32_t num_states;
  int64_t num_arcs;
  const int64_t *row_offsets; /* [num_states + 1] */
  const int32_t *ilabels;     /* [num_arcs] */
  const int32_t *olabels;     /* [num_arcs] */
  const int32_t *next_states; /* [num_arcs] */
  const double *weights;      /* [num_arcs] */
  const uint8_t *is_final;    /* [num_states] */
  const double *final_costs;  /* [num_states], read only where is_final */
  int32_t num_emitting_labels; /* max ilabel (fst.py:141-145) */
} orc_graph;

/* DecoderConfig (decoder.py:33-48). */
typedef struct orc_config {
  double beam;
  int32_t max_active;
  int32_t max_eps;
  int32_t partial_every;
  int32_t endpoint_silence_frames;
  int32_t silence_ilabel;
} orc_config;

/* BiasingContext (biasing.py:86-117): strictly increasing arc ids + discount. */
typedef struct orc_context {
  const int64_t *arc_indices;
  int64_t k;
  double discount;
} orc_context;

enum { ORC_IDLE = 0, ORC_DECODING = 1, ORC_ENDPOINTED = 2, ORC_FINISHED = 3 };
enum {
  ORC_OK = 0,
  ORC_ERR_DEAD = 1,   /* "decode failure, no active tokens" */
  ORC_ERR_WIDTH = 2,  /* frame width != emitting-label count */
  ORC_ERR_STATUS = 3, /* advance/finalize in a wrong status */
  ORC_ERR_CAPACITY = 4,
  ORC_ERR_ALLOC = 5
};
enum { ORC_PARTIAL = 0, ORC_FINAL = 1 };

typedef struct orc_hyp {
  double cost;
  int64_t frame;
  int32_t kind;
  int32_t fallback;
  int64_t hits;
  int64_t words_off;
  int64_t n_words;
} orc_hyp;

typedef struct orc_channel orc_channel;

typedef struct orc_channel_info {
  int32_t status;
  int32_t fresh;
  int64_t frame_index;
  int64_t total_frames;
  int64_t utterance_index;
  int64_t trailing_silence;
  int64_t eps_truncations;
  int64_t num_active;
  int64_t store_len;
  /* per-frame work counters of the last advance (SURVEY §8d algorithmic bytes) */
  int64_t tok_expansions;
  int64_t emit_arcs;
  int64_t eps_arcs;
} orc_channel_info;

orc_channel *orc_channel_new(const orc_graph *g);
void orc_channel_free(orc_channel *ch);
void orc_channel_get_info(const orc_channel *ch, orc_channel_info *out);
void orc_channel_set_status(orc_channel *ch, int32_t status);
void orc_channel_set_trailing_silence(orc_channel *ch, int64_t v);

int orc_advance(orc_channel *ch, const orc_graph *g, const orc_context *ctx,
                const orc_config *cfg, const double *row, int64_t width);
/* Token table sorted by state: writes up to cap entries, returns count. */
int64_t orc_tokens(const orc_channel *ch, int32_t *states, double *costs, int64_t *hits,
                   int64_t cap);
int orc_partial(orc_channel *ch, orc_hyp *hyp, int32_t *words, int64_t words_cap);
int orc_finalize(orc_channel *ch, const orc_graph *g, orc_hyp *hyp, int32_t *words,
                 int64_t words_cap);
/* _decode_one (decoder.py:474-501) over a [T, width] row-major score matrix. */
int orc_decode_stream(orc_channel *ch, const orc_graph *g, const orc_context *ctx,
                      const orc_config *cfg, const double *scores, int64_t T, int64_t width,
                      orc_hyp *hyps, int64_t hyp_cap, int64_t *n_hyps, int32_t *words,
                      int64_t words_cap, int64_t *n_words);

#ifdef __cplusplus
}
#endif
#endif
