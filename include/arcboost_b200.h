/*
 * arcboost-b200 C ABI — batched biased token-passing Viterbi on sm_100a.
 *
 * This is the drop-in boundary for the reference decode path
 * (/root/reference/pkg/src/arcboost/decoder.py).  The reference has no FFI;
 * its boundary is the Python API re-exported from arcboost/__init__.py:21-35.
 * Each entry point below names the reference interface it replaces; the
 * Python package paper_2306_15685_b200 binds these through ctypes and
 * re-exposes the reference names.
 *
 * Conventions: every function returns 0 on success or an AB_ERR_* code; the
 * message of the last failure on the calling thread is ab_last_error().
 * Host input buffers are copied; the caller keeps ownership.  Device memory
 * is owned by the library.  One decoder per device; calls on one decoder must
 * be serialised by the caller (different decoders may run on different host
 * threads), and so must context registration / release on one graph (the
 * context store and its slack scratch are per graph).  No torch types cross
 * this boundary.
 */
#ifndef ARCBOOST_B200_H
#define ARCBOOST_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  AB_OK = 0,
  AB_ERR_INVALID = 1,      /* bad argument (ValueError on the Python side) */
  AB_ERR_CUDA = 2,         /* CUDA runtime failure / no device */
  AB_ERR_DEAD = 3,         /* "decode failure, no active tokens" (decoder.py:419-420, 438-439) */
  AB_ERR_STATUS = 4,       /* lifecycle misuse (decoder.py:352-353, 430-433) */
  AB_ERR_CAPACITY = 5,     /* a device capacity (token table, arena, output) was exceeded */
  AB_ERR_UNKNOWN_CTX = 6,  /* UnknownContextError (biasing.py:27) */
  AB_ERR_WIDTH = 7,        /* frame width != emitting-label count (decoder.py:354-359) */
  AB_ERR_PARSE = 8,        /* FstParseError (fst.py:24): malformed graph text */
  AB_ERR_STRUCTURE = 9,    /* FstStructureError (fst.py:28) */
  AB_ERR_SCORE_FORMAT = 10 /* ScoreFormatError (scores.py:15) */
};

enum { AB_IDLE = 0, AB_DECODING = 1, AB_ENDPOINTED = 2, AB_FINISHED = 3 };
enum { AB_PARTIAL = 0, AB_FINAL = 1 };
enum { AB_F32 = 0, AB_F64 = 1 };
/* ab_decode modes */
enum {
  AB_MODE_ADVANCE = 0, /* advance_frame only, T frames (decoder.py:341-411) */
  AB_MODE_STREAM = 1   /* _decode_one: partial cadence, endpointing, final (decoder.py:474-501) */
};
/* context lookup representation (ab_context_register mode):
   LIST    the arc ids as a hash set in HBM, behind a Bloom filter in shared
           memory when k <= 2048
   BITSET  one bit per arc (by device record position) in HBM
   LABELS  one bit per output label in shared memory; only valid (and only
           chosen by AUTO) when the context is exactly the set of arcs whose
           olabel lies in some label set, e.g. single-word entities */
enum { AB_CTX_AUTO = 0, AB_CTX_LIST = 1, AB_CTX_BITSET = 2, AB_CTX_LABELS = 3 };
/* device limits: distinct tokens per channel-frame, hashed-table slots; the
   epsilon-round cap is not limited (any int32, negative = no rounds, as
   decoder.py:263 `rounds < max_epsilon_expansion`) */
enum { AB_MAX_TOKENS = 131072, AB_MAX_HASH_SLOTS = 4194304, AB_MAX_EPSILON_ROUNDS = 2147483647 };

typedef struct ab_graph ab_graph;
typedef struct ab_fst ab_fst; /* a parsed graph on the host (state-major CSR) */
typedef struct ab_scores ab_scores; /* a parsed score matrix on the host */
typedef struct ab_decoder ab_decoder;

/* DecoderConfig (decoder.py:33-48). */
typedef struct ab_config {
  double beam;
  int32_t max_active;
  int32_t max_epsilon_expansion;
  int32_t partial_every;
  int32_t endpoint_silence_frames;
  int32_t silence_ilabel;
  /* AB_CFG_EXACT: relax every candidate, as the reference does, so len(store)
     and eps_truncations count the applications of candidates that cannot
     survive the frame too.  Default (0): candidates provably outside the
     frame's survivors are dropped at expansion (same surviving tokens, costs,
     hypotheses; those two counters then count relaxed candidates only). */
  int32_t flags;
} ab_config;

#define AB_CFG_EXACT 1

/* Device capacities per channel; 0 selects a default derived from the graph. */
typedef struct ab_capacity {
  int64_t table_slots;   /* token table: >= num_states (or 0 when the budget allows: 20 B per
                            state and channel, AB_DIRECT_TABLE_GB or 60% of free HBM) selects
                            a direct table (slot = state); fewer slots a hashed table
                            (rounded up to a power of two, <= AB_MAX_HASH_SLOTS) */
  int64_t frontier_rows; /* epsilon-frontier log rows per frame */
  int64_t arena_records; /* emission records per utterance */
  int64_t path_words;    /* longest hypothesis path */
} ab_capacity;

/* Channel fields (decoder.py:119-139) mirrored between host and device. */
typedef struct ab_channel_info {
  int32_t status;
  int32_t fresh;
  int64_t frame_index;
  int64_t total_frames;
  int64_t utterance_index;
  int64_t trailing_silence;
  int64_t eps_truncations;
  int32_t context;     /* context handle, -1 = unbiased */
  int32_t num_active;  /* len(_states) */
  int64_t store_len;   /* len(store) */
  int32_t error;       /* last device error code for this channel */
  int32_t cut_redos;   /* frames redone without the expansion-time cutoff (its hint was
                          below the frame's cutoff; see ab_config.flags) */
  /* work counters accumulated by the device: token expansions,
     emitting arcs, epsilon arcs */
  uint64_t tok_expansions;
  uint64_t emit_arcs;
  uint64_t eps_arcs;
} ab_channel_info;

/* One hypothesis as produced on the device (Hypothesis, decoder.py:110-116).
   Words are prefix-shared: the hypothesis' words are the first `shared` words
   of the channel's previous hypothesis followed by n_words - shared words
   stored at words_off in the batch word pool. */
typedef struct ab_hyp {
  double cost;
  int64_t frame;
  int32_t kind;
  int32_t fallback;
  int32_t hits; /* boosted arcs on the hypothesis path */
  int32_t shared;
  int32_t n_words;
  int32_t pad_;
  int64_t words_off;
} ab_hyp;

/* One batched decode call (decode_batch, decoder.py:504-526). */
typedef struct ab_decode_args {
  int32_t n;                 /* channels in the batch */
  const int32_t *channels;   /* [n] channel slots (host) */
  const int32_t *frames;     /* [n] frames per channel (host) */
  const int64_t *score_offsets; /* [n] element offset of each channel's [T, L] block */
  const void *scores;        /* f32 or f64 [*, L] rows */
  int32_t scores_on_device;  /* 1: device pointer; 0: host pointer (copied inside the call) */
  int32_t scores_dtype;      /* AB_F32 / AB_F64 */
  int32_t width;             /* L, must equal the graph's emitting-label count */
  int32_t mode;              /* AB_MODE_* */
  ab_config config;
  void *stream;              /* cudaStream_t, NULL = library stream */
} ab_decode_args;

const char *ab_last_error(void);
int ab_device_count(int32_t *count);

/* Re-reads the environment knobs (AB_CUT_HINT_MIN, AB_CUT_HINT_EXTRA: the
   expansion-time cutoff's hint margin, see ab_config.flags). */
void ab_reload_env(void);

/* build_csr (fst.py:165-191) → device CSR split into emitting / epsilon SoA. */
int ab_graph_create(int32_t device, int32_t start, int32_t num_states, int64_t num_arcs,
                    const int64_t *row_offsets, const int32_t *ilabels, const int32_t *olabels,
                    const int32_t *next_states, const double *weights, int32_t num_finals,
                    const int32_t *final_states, const double *final_costs, ab_graph **out);
void ab_graph_destroy(ab_graph *g);
/* num_emitting_labels (fst.py:141-145) and storage facts. */
int ab_graph_query(const ab_graph *g, int32_t *num_emitting_labels, int32_t *weights_f32,
                   int64_t *device_bytes);

/* The expansion-time cutoff's epsilon slack of a context (handle -1: the
   unbiased graph): the most an epsilon path lowers a token's cost under its
   weighting, and the number of set bits in the Bloom filter of the states it
   applies to (negated when the slack bounds paths of at most 64 epsilon arcs
   only: a negative epsilon cycle or a longer chain). */
int ab_context_slack(const ab_graph *g, int32_t handle, double *slack, int32_t *neg_states);

/* BiasingContext (biasing.py:86-117) → device context store entry.  arc_indices
   must be strictly increasing and non-negative (indices >= num_arcs never match).
   mode: AB_CTX_AUTO (LABELS when the set is exactly the arcs of some output
   labels, LIST up to 2048 arcs, else BITSET) or a forced representation.  Also
   computes the context's epsilon slack for the expansion-time cutoff (host,
   from the negative epsilon arcs backwards). */
int ab_context_register(ab_graph *g, const int64_t *arc_indices, int64_t k, double discount,
                        int32_t mode, int32_t *handle);
/* representation the context store chose for a handle (AB_CTX_LIST/BITSET/LABELS) */
int ab_context_mode(const ab_graph *g, int32_t handle, int32_t *mode);
int ab_context_release(ab_graph *g, int32_t handle);

int ab_decoder_create(ab_graph *g, const ab_capacity *cap, int32_t max_channels,
                      ab_decoder **out);
void ab_decoder_destroy(ab_decoder *d);
int ab_decoder_query(const ab_decoder *d, ab_capacity *cap, int64_t *device_bytes);

/* init_channel (decoder.py:162-174): fresh IDLE channel in slot ch. */
int ab_channel_init(ab_decoder *d, int32_t ch, int32_t context);
/* switch_context (decoder.py:177-193); rejects a mid-utterance switch. */
int ab_channel_set_context(ab_decoder *d, int32_t ch, int32_t context);
int ab_channel_get(ab_decoder *d, int32_t ch, ab_channel_info *info);
/* Host-side lifecycle edits (status / trailing_silence / fresh) pushed to the device. */
int ab_channel_put(ab_decoder *d, int32_t ch, const ab_channel_info *info);
/* Batched forms for large channel counts (one transfer each). */
int ab_channels_init(ab_decoder *d, int32_t n, const int32_t *slots, const int32_t *contexts);
int ab_channels_set_context(ab_decoder *d, int32_t n, const int32_t *slots,
                            const int32_t *contexts);
int ab_channels_get(ab_decoder *d, int32_t n, const int32_t *slots, ab_channel_info *infos);
/* Active token table: states / costs / hits / backpointers (device emission-record
   id of the token's newest word, -1 = none); any pointer may be NULL.  Returns
   the count in *n.  (Token fields, decoder.py:58-62.) */
int ab_channel_tokens(ab_decoder *d, int32_t ch, int32_t *states, double *costs, int32_t *hits,
                      int32_t *backpointers, int32_t cap, int32_t *n);

/* advance_frame × T / _decode_one for a batch; results stay on the device. */
int ab_decode(ab_decoder *d, const ab_decode_args *args);
/* Results of the last ab_decode: per batch entry the hypothesis count and the
   first device error (0 = none) plus the frame index at which it occurred. */
int ab_read_results(ab_decoder *d, int32_t *n_hyps, int32_t *errors, ab_hyp *hyps,
                    int32_t hyp_stride, int32_t *words, int64_t words_cap, int64_t *words_used);
/* partial_hypothesis (decoder.py:414-423) / finalize (decoder.py:426-460) for one channel. */
int ab_partial(ab_decoder *d, int32_t ch, ab_hyp *hyp, int32_t *words, int32_t words_cap);
int ab_finalize(ab_decoder *d, int32_t ch, ab_hyp *hyp, int32_t *words, int32_t words_cap);
/* Device time of the last ab_decode's decode kernels in milliseconds (CUDA
   events on the launching stream) and the number of kernels it launched. */
int ab_last_kernel_ms(ab_decoder *d, float *ms);
int ab_last_launch_count(ab_decoder *d, int32_t *launches);

/* Paper Alg. 1 (biasing.py:174-285 find_boost_arcs / compile_context): the
   arc indices a context boosts for a batch of word-label entities over the
   host CSR (row_offsets[num_states + 1], olabels / next_states[num_arcs]).
   Entity e is labels[ent_offsets[e] .. ent_offsets[e + 1]).  ent_status[e] =
   1 compiled, 0 unmatched, -1 invalid (empty or containing epsilon).  The
   sorted union is written to out_arcs (at most out_cap; *n_out = its size,
   call again with a larger buffer if *n_out > out_cap).  CPU, num_threads
   threads (0 = all). */
/* Graph ingest (fst.py:165-275 parse_text_fst + build_csr + _fingerprint):
   OpenFst-style text -> host CSR.  ab_fst_parse parses a text buffer;
   ab_fst_load parses a file and, with use_cache, reads / writes a binary
   cache at cache_path (reused while the source's size and mtime match).
   num_states_hint < 0 = none.  AB_ERR_PARSE / AB_ERR_STRUCTURE carry the
   reference's messages.  ab_fst_arrays copies the CSR out (arrays sized from
   ab_fst_info); ab_graph_create_from_fst uploads it directly. */
int ab_fst_parse(const char *text, int64_t len, int64_t num_states_hint, ab_fst **out);
int ab_fst_load(const char *path, int64_t num_states_hint, int32_t use_cache, const char *cache_path,
                int32_t *cache_hit, ab_fst **out);
int ab_fst_info(const ab_fst *f, int32_t *start, int64_t *num_states, int64_t *num_arcs,
                int32_t *num_finals, char *fingerprint65);
int ab_fst_arrays(const ab_fst *f, int64_t *row_offsets, int32_t *ilabels, int32_t *olabels,
                  int32_t *next_states, double *weights, int32_t *final_states, double *final_costs);
void ab_fst_destroy(ab_fst *f);
int ab_graph_create_from_fst(int32_t device, const ab_fst *f, ab_graph **out);
/* Score ingest (scores.py:52-96 parse_score_matrix / load_score_matrix):
   the text format into a host [num_frames, num_ilabels] f64 matrix with the
   reference's checks; AB_ERR_SCORE_FORMAT carries its messages. */
int ab_scores_parse(const char *text, int64_t len, ab_scores **out);
int ab_scores_info(const ab_scores *s, int64_t *num_frames, int64_t *num_ilabels, double *frame_duration);
int ab_scores_copy(const ab_scores *s, double *costs);
void ab_scores_destroy(ab_scores *s);
int ab_compile_context(int32_t num_states, int64_t num_arcs, const int64_t *row_offsets,
                       const int32_t *olabels, const int32_t *next_states, int32_t n_entities,
                       const int64_t *ent_offsets, const int32_t *labels,
                       int32_t max_epsilon_depth, int32_t num_threads, int64_t *out_arcs,
                       int64_t out_cap, int64_t *n_out, int32_t *ent_status);

/* Run scoring (metrics.py:26-83 align / compute_wer), words as integer ids.
   ab_align: the minimum-edit-distance alignment with the reference's
   backtrace tie order (match, substitution, deletion, insertion); kind[i] in
   {0 match, 1 substitution, 2 deletion, 3 insertion}, ref_pos / hyp_pos -1
   where absent.  *n_ops is the full count (<= nr + nh); at most cap ops are
   written.  ab_edit_distances: the edit distance of each of n pairs (words
   ref[ref_off[p]:ref_off[p+1]] vs hyp[...]), pairs over num_threads host
   threads (0 = all). */
int ab_align(const int32_t *ref, int64_t nr, const int32_t *hyp, int64_t nh, int8_t *kind,
             int32_t *ref_pos, int32_t *hyp_pos, int64_t cap, int64_t *n_ops);
int ab_edit_distances(int64_t n, const int64_t *ref_off, const int32_t *ref, const int64_t *hyp_off,
                      const int32_t *hyp, int32_t num_threads, int64_t *dist);

/* Synthetic scores on the device (synth.py:69-75, 156-195; the benchmark's
   default_rng([seed, channel]).uniform streams): n_streams numpy PCG64
   streams, streams[4*s..4*s+3] = {state >> 64, state & (2^64-1), inc >> 64,
   inc & (2^64-1)} as numpy's bit_generator.state reports them; writes
   out[s * values_per_stream + k] = offset + (low + (high - low) * u_k), u_k the
   k-th next_double of stream s, bit-identical to numpy, as f32 (AB_F32,
   rounded to nearest) or f64, into device memory.  Synchronous on stream. */
int ab_scores_generate(int32_t device, const uint64_t *streams, int32_t n_streams, int64_t values_per_stream,
                       double low, double high, double offset, int32_t dtype, void *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif
