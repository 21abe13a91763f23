/*
 * tbeam_b200.h -- C-ABI boundary of the B200-native batched Transducer beam
 * search (ALSD++ / AES++ / label-looping greedy, RNN-T and TDT, n-gram LM
 * shallow fusion).
 *
 * This header is the drop-in boundary for the reference decoder API in
 * /root/reference/proj/include/tbeam/decoder.hpp.  Each entry point names the
 * reference interface it replaces:
 *
 *   tbeam_decode(cfg.algo = GREEDY)   <- tbeam::greedy_batched   decoder.hpp:75-76
 *   tbeam_decode(cfg.algo = ALSD)     <- tbeam::alsd_pp          decoder.hpp:79
 *   tbeam_decode(cfg.algo = AES)      <- tbeam::aes_pp           decoder.hpp:83
 *   tbeam_decode_config               <- tbeam::DecodeConfig     decoder.hpp:23-42
 *                                        + tbeam::FusionConfig   fusion.hpp:19-24
 *                                        + tbeam::HashParams     hyp_store.hpp:15-18
 *   tbeam_model_dims / _weights       <- tbeam::EmissionModel    model.hpp:62-74
 *                                        (the per-row virtual score_row call is
 *                                        replaced by device-resident weights +
 *                                        encoder frames)
 *   tbeam_set_lm_arpa                 <- tbeam::NGramLm::parse_arpa_text
 *                                                                ngram_lm.hpp:38-42
 *   tbeam_results                     <- tbeam::DecodeResult     decoder.hpp:52-70
 *   tbeam_status codes                <- std::invalid_argument / CapacityError /
 *                                        ParseError / ValidationError  types.hpp:29-52
 *
 * Plain C types only: pointers, sizes, POD structs.  No torch types.
 * Ownership: the caller owns every host buffer it passes in; the context owns
 * every device buffer it allocates.  A context is bound to one CUDA device and
 * is thread-compatible (one context per thread).
 */
#ifndef TBEAM_B200_H_
#define TBEAM_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TBEAM_B200_ABI_VERSION 1

/* ---- status codes (reference exception taxonomy, types.hpp:29-52) -------- */
typedef enum {
    TBEAM_OK = 0,
    TBEAM_INVALID_ARGUMENT = 1, /* std::invalid_argument (decoder.cpp:16-38)   */
    TBEAM_CAPACITY = 2,         /* tbeam::CapacityError                         */
    TBEAM_PARSE = 3,            /* tbeam::ParseError (ARPA text)                */
    TBEAM_VALIDATION = 4,       /* tbeam::ValidationError                       */
    TBEAM_CUDA = 5,             /* CUDA runtime / driver failure                */
    TBEAM_UNSUPPORTED = 6       /* build or device lacks a required feature     */
} tbeam_status;

/* ---- algorithms, fusion modes (fusion.hpp:13-17) -------------------------- */
enum { TBEAM_ALGO_GREEDY = 0, TBEAM_ALGO_ALSD = 1, TBEAM_ALGO_AES = 2 };
enum { TBEAM_BLANK_OMIT = 0, TBEAM_BLANK_SCORED = 1 };   /* BlankMode  */
enum { TBEAM_PRUNE_EARLY = 0, TBEAM_PRUNE_LATE = 1 };    /* PruneMode  */
enum { TBEAM_MERGE_LOGSUMEXP = 0, TBEAM_MERGE_MAX = 1 };
enum { TBEAM_PRED_STATELESS = 0, TBEAM_PRED_LSTM = 1 };
/* Precision of the decode GEMMs (joint, LSTM gates / projection, encoder
 * projection).  FP32: scores within 1e-4 of the fp64 reference -- the tensor
 * cores on operands split into three bf16 planes (x = x0 + x1 + x2 exactly,
 * six plane products, one fp32 TMEM accumulator per 64-wide k-block summed in
 * fp64); env TBEAM_FP32_SIMT=1 selects the CUDA-core FFMA kernels instead.
 * BF16: bf16 operands, fp32 accumulation (bound 4e-5 x frames decoded).
 * Hypothesis scores, normalisers and LM values are fp64 in both. */
enum { TBEAM_PREC_FP32 = 0, TBEAM_PREC_BF16 = 1 };

#define TBEAM_MAX_DURATIONS 8
#define TBEAM_NUM_COUNTERS 5 /* frames, scoring_rounds, scored_slots,
                                lm_token_queries, lm_vocab_queries
                                (tbeam::Counters, decoder.hpp:44-50) */

/* DecodeConfig + FusionConfig + HashParams, field for field, plus the
 * B200 additions (algo, merge mode, AES slot-quirk compat flag). */
typedef struct {
    int32_t algo;                     /* TBEAM_ALGO_*                          */
    int32_t beam;                     /* DecodeConfig::beam (4)                */
    int32_t max_symbols_per_frame;    /* ALSD++/greedy rounds per frame (10)   */
    int32_t aes_expansions_per_frame; /* AES++ token rounds per frame (2)      */
    int32_t max_len;                  /* U_max (256)                           */
    int32_t return_nbest;             /* (1)                                   */
    int32_t aes_prefix_search;        /* (1)                                   */
    double lm_weight;                 /* FusionConfig::lambda (0)              */
    int32_t blank_mode;               /* TBEAM_BLANK_* (omit)                  */
    int32_t prune_mode;               /* TBEAM_PRUNE_* (late)                  */
    int32_t eos_enabled;              /* (0)                                   */
    int32_t merge_mode;               /* TBEAM_MERGE_* (logsumexp = reference) */
    uint64_t hash_base;               /* HashParams::base (1000003)            */
    uint64_t hash_modulus;            /* HashParams::modulus (2^61-1)          */
    /* 1 = reproduce the shipped aes_pp's stale per-slot donated[] flag
     * (decoder.cpp:124,:145,:227,:245).  0 = canonical AES++
     * (reference_beam(kAes), reference_decoder.cpp:232-234). */
    int32_t aes_slot_donated_quirk;
    int32_t reserved[7];
} tbeam_decode_config;

/* Synthetic transducer shape.  Emission row layout follows the reference:
 * V real tokens, blank id = V (last).  TDT adds a duration head. */
typedef struct {
    int32_t vocab_size;    /* V                                               */
    int32_t enc_dim;       /* D: encoder frame width                          */
    int32_t joint_dim;     /* J                                               */
    int32_t pred_kind;     /* TBEAM_PRED_*                                    */
    int32_t context_order; /* n (stateless)                                   */
    int32_t lstm_hidden;   /* H (LSTM)                                        */
    int32_t emb_dim;       /* E (LSTM input embedding)                        */
    int32_t num_durations; /* 0 = RNN-T; >0 = TDT                             */
    int32_t durations[TBEAM_MAX_DURATIONS]; /* ascending, e.g. {0,1,2,3,4}    */
    int32_t precision;     /* TBEAM_PREC_*: operand precision of the GEMMs    */
    int32_t reserved[3];
} tbeam_model_dims;

/* Host fp32 weights, row-major.  Unused pointers may be NULL.
 *   enc_proj[b,t]  = w_enc . enc[b,t] + b_enc                      [J]
 *   stateless:  pred = b_pred + (1/n) sum_i pred_table[w_i]         [J]
 *               (BOS padding uses row V)
 *   LSTM:       gates = w_ih . emb[tok] + w_hh . h + b_lstm  (i,f,g,o)
 *               c' = sig(f) c + sig(i) tanh(g);  h' = sig(o) tanh(c')
 *               pred = w_pred . h' + b_pred; start state = step(0,0,emb[V])
 *   z = tanh(enc_proj + pred);  token logits = w_out . z + b_out   [V+1]
 *   TDT:        duration logits = w_dur . z + b_dur                 [ND]   */
typedef struct {
    const float* w_enc;      /* [J, D]     */
    const float* b_enc;      /* [J]        */
    const float* pred_table; /* [V+1, J]   */
    const float* b_pred;     /* [J]        */
    const float* emb;        /* [V+1, E]   */
    const float* w_ih;       /* [4H, E]    */
    const float* w_hh;       /* [4H, H]    */
    const float* b_lstm;     /* [4H]       */
    const float* w_pred;     /* [J, H]     */
    const float* w_out;      /* [V+1, J]   */
    const float* b_out;      /* [V+1]      */
    const float* w_dur;      /* [ND, J]    */
    const float* b_dur;      /* [ND]       */
} tbeam_model_weights;

/* DecodeResult (decoder.hpp:52-70) flattened into caller-owned arrays.
 * Per stream b: nbest_count[b] <= nbest entries, descending score, distinct
 * transcripts.  Entry (b, r): lengths[b*nbest+r] tokens in
 * tokens[(b*nbest+r)*max_len ...]; frames[] = encoder frame each token was
 * emitted at (alignment); durations[] = TDT duration of each token (0 for
 * RNN-T).  counters[b*5 + i] = tbeam::Counters fields. */
typedef struct {
    int32_t batch;
    int32_t nbest;
    int32_t max_len;
    int32_t* nbest_count; /* [B]                 */
    int32_t* lengths;     /* [B, nbest]          */
    double* scores;       /* [B, nbest]          */
    int32_t* tokens;      /* [B, nbest, max_len] */
    int32_t* frames;      /* [B, nbest, max_len] (may be NULL) */
    int32_t* durations;   /* [B, nbest, max_len] (may be NULL) */
    uint64_t* counters;   /* [B, 5]              (may be NULL) */
} tbeam_results;

typedef struct tbeam_ctx tbeam_ctx;

/* Defaults of decoder.hpp:23-42 / fusion.hpp:19-24 / hyp_store.hpp:15-18. */
void tbeam_decode_config_init(tbeam_decode_config* cfg);

/* Context on CUDA device `device`.  Fails with TBEAM_UNSUPPORTED when the
 * device is not sm_100 or the sm_100a kernels are missing from the build. */
tbeam_status tbeam_create(int device, tbeam_ctx** out);
tbeam_status tbeam_destroy(tbeam_ctx* ctx);

/* Upload weights (converted to the operand precision on device). */
tbeam_status tbeam_set_model(tbeam_ctx* ctx, const tbeam_model_dims* dims,
                             const tbeam_model_weights* weights);

/* Parse ARPA text (NGramLm::parse_arpa_text semantics, ngram_lm.cpp:52-318)
 * against the ASR token table and upload the frozen trie to the device.
 * `tokens` holds vocab_size NUL-terminated strings (id = index). */
tbeam_status tbeam_set_lm_arpa(tbeam_ctx* ctx, const char* arpa_text, size_t len,
                               const char* const* tokens, int32_t vocab_size,
                               int32_t strict);
tbeam_status tbeam_clear_lm(tbeam_ctx* ctx);
/* Host-only ARPA validation (no GPU needed): parses like tbeam_set_lm_arpa and
 * reports order, node count, edge count, <unk>-mapped count in out[4]. */
tbeam_status tbeam_lm_parse_check(const char* arpa_text, size_t len,
                                  const char* const* tokens, int32_t vocab_size,
                                  int32_t strict, int64_t out[4]);
/* Host-only inspection of the frozen trie the device queries walk (tests and
 * tooling; no GPU).  Call with NULL arrays to get the sizes in out[4] (order,
 * node count, edge count, initial state); then again with arrays of those
 * sizes: per node prob/backoff (ln; NaN prob = implicit context node),
 * suffix link, depth, child edge range [cbeg, cend); per edge the internal
 * token and child node; remap[vocab_size] = internal id of each ASR token
 * (-1 = none).  Internal ids: ASR tokens 0..V-1, <s> V, </s> V+1, <unk> V+2. */
tbeam_status tbeam_lm_export(const char* arpa_text, size_t len,
                             const char* const* tokens, int32_t vocab_size,
                             int32_t strict, int64_t out[4], double* prob,
                             double* backoff, int32_t* suffix, int32_t* depth,
                             int32_t* cbeg, int32_t* cend, int32_t* etok,
                             int32_t* enode, int32_t* remap);
/* LM statistics: order, node count, edge count, <unk>-mapped token count. */
tbeam_status tbeam_lm_info(tbeam_ctx* ctx, int64_t out[4]);

/* Decode `batch` streams.  enc is [batch, max_frames, enc_dim] fp32 (it must
 * hold batch * max_frames * dims.enc_dim floats; enc_dim is the model's), host
 * memory (copied in on `stream`) or device memory (enc_on_device = 1).
 * lengths[b] in [1, max_frames] (host array).  Results land in `res`
 * (host, caller-owned).  Synchronous on return.  stream may be NULL. */
tbeam_status tbeam_decode(tbeam_ctx* ctx, const tbeam_decode_config* cfg,
                          const float* enc, int32_t enc_on_device,
                          const int32_t* lengths, int32_t batch,
                          int32_t max_frames, tbeam_results* res, void* stream);

/* Pipelined serving from HOST buffers (the same decode as tbeam_decode, split
 * in two so consecutive batches overlap):
 *   tbeam_stage_inputs  copies a batch's encoder frames and lengths (pinned
 *                       host memory lets the copy run asynchronously) into
 *                       the next of two device input slots on the context's
 *                       copy stream and returns at once;
 *   tbeam_decode_staged decodes the oldest staged batch on `stream` (behind
 *                       its copy) and fetches its results like tbeam_decode.
 * Staging batch i+1 before decoding batch i overlaps its H2D copy with batch
 * i's decode.  At most two batches are staged ahead (TBEAM_INVALID_ARGUMENT
 * otherwise); a slot is reused only after the decode that read it returned.
 * The host buffers must stay unchanged until tbeam_decode_staged of their
 * batch returns. */
tbeam_status tbeam_stage_inputs(tbeam_ctx* ctx, const float* enc_host,
                                const int32_t* lengths, int32_t batch,
                                int32_t max_frames);
tbeam_status tbeam_decode_staged(tbeam_ctx* ctx, const tbeam_decode_config* cfg,
                                 tbeam_results* res, void* stream);

/* Device-resident variant for benchmarking: runs the whole decode on
 * `stream` without any host synchronisation or copies.  enc_dev and
 * lengths_dev are device pointers; results stay in the context's device
 * buffers until tbeam_fetch_results.  Call tbeam_prepare first with the same
 * (cfg, batch, max_frames) to allocate and capture the CUDA graph. */
tbeam_status tbeam_prepare(tbeam_ctx* ctx, const tbeam_decode_config* cfg,
                           int32_t batch, int32_t max_frames);
tbeam_status tbeam_decode_device(tbeam_ctx* ctx, const float* enc_dev,
                                 const int32_t* lengths_dev, void* stream);
tbeam_status tbeam_fetch_results(tbeam_ctx* ctx, tbeam_results* res, void* stream);

/* Instrumented decode for measurement (not the timed path): runs the same
 * kernels as tbeam_decode_device but host-driven, bracketing every launch
 * with CUDA events on `stream`.  Per kernel family f (0 enc_proj, 1 init,
 * 2 joint, 3 select (+ prediction-state gather), 4 LSTM gate GEMM, 5 LSTM
 * projection GEMM, 6 finalize):
 * ms_out[f] = summed device time, launches_out[f] = launch count.  Also
 * fills rows_out[0] = scored joint rows, rows_out[1] = rounds.  Returns the
 * number of families (7) or -1. */
int32_t tbeam_profile_decode(tbeam_ctx* ctx, const float* enc_dev,
                             const int32_t* lengths_dev, void* stream,
                             double* ms_out, int64_t* launches_out,
                             int64_t* rows_out);

/* Kernel launches issued by the most recent decode, counted on the device
 * (per kernel family).  out[0] = total; returns number of entries written. */
int32_t tbeam_launch_stats(tbeam_ctx* ctx, int64_t* out, int32_t cap);

/* Execution mode: 1 = whole decode loop in one CUDA graph with a
 * conditional WHILE node (default); 0 = host-driven loop over a captured
 * per-round graph (debug). */
tbeam_status tbeam_set_graph_mode(tbeam_ctx* ctx, int32_t mode);

/* Last error message of the calling thread ("" when none). */
const char* tbeam_last_error(void);
int32_t tbeam_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TBEAM_B200_H_ */
