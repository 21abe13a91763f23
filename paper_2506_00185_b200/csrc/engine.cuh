// Device-side data layout of the B200 batched Transducer beam search.
//
// Everything a decode needs lives in HBM for the whole decode; the per-round
// loop never touches the host.  Layout (B streams, K beam, S = B*K slots,
// R = V+1 emission columns with the blank last, ND TDT durations):
//
//   per stream [B]          T_b, t (current frame), r (round in frame),
//                           done, steps, counters[5]
//   per slot   [S]          score f64, len, hash u64, last, f (frame of the next
//                           emission), tnode (newest token node), lm_state,
//                           donated (per hypothesis) + slot_donated (aes_pp quirk)
//   pred state [2][S][...]  parity double buffer: stateless window [n] or LSTM
//                           h[H], c[H]; pred projection [J] fp32
//   token trie [cols][S]    tok i32, prev node i32, dur i8: one node per emitted
//                           token (column = round), frame[cols][B] = t of the
//                           round -- the paper's backlink trie (§2.1 Fig. 1)
//                           indexed by emission, so a backtrace walks U nodes
//   joint partials          per (slot, N-tile): max, sum-exp, top-K
//                           (raw, idx, logit, lm); blank logit, duration logits
//   active lists [2][S]     compacted rows to score next round (parity g&1)
//
// Reference counterparts: BatchedBeamHyps (hyp_store.hpp:52-136),
// BeamEngine::run_lane locals (decoder.cpp:120-141), Counters (decoder.hpp:44-50).
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace tbeam_dev {

__host__ __device__ inline int part_stride(int K) { return 4 + 4 * K; }

constexpr int kMaxBeam = 32;
constexpr int kMaxDur = 8;
constexpr int kMaxOrder = 8;  // LM backoff chain held in registers: n-gram order <= kMaxOrder + 1 (checked at load)
constexpr double kLogZeroFloor = -1e9;
constexpr std::uint64_t kMersenne61 = (std::uint64_t{1} << 61) - 1;

struct DevModel {
    int V, R, D, J, H, E, ND, n, pred_kind, prec;
    int durations[kMaxDur];
    int di0;  // index of duration 0 or -1
    const float* w_enc;      // [J, D]
    const float* b_enc;      // [J]
    const float* table;      // [R, J] stateless
    const float* b_pred;     // [J]
    const float* xtab;       // [R, 4H] LSTM input table (W_ih . emb + b)
    const float* w_hh;       // [4H, H]  (fp32 mode)
    const float* w_pred;     // [J, H]
    const float* w_out;      // [R + ND, J] token rows then duration rows
    const float* b_out;      // [R + ND]
    const __nv_bfloat16* w_enc16;  // bf16 operand copies (precision = bf16)
    const __nv_bfloat16* w_hh16;
    const __nv_bfloat16* w_pred16;
    const __nv_bfloat16* w_out16;  // [Npad, J]
    const float* h0;    // [H]  LSTM start state
    const float* c0;    // [H]
    const float* pred0; // [J]  start prediction output
};

struct DevLm {
    int present;
    int order;
    int V;
    int initial;
    const double* prob;     // NaN = implicit context node
    const double* backoff;
    const int* suffix;
    const int* depth;
    const int* cbeg;
    const int* cend;
    const int* etok;        // children sorted by token per node
    const int* enode;
    const int* remap;       // [V] ASR id -> internal id or -1
    const float* uni;       // [V] root child prob or NaN
    const int* root;        // [n_root] dense root children: internal id -> node or -1
    int n_root;
    double unk_prob;        // -inf when no <unk> unigram
};

struct DevCfg {
    int algo, K, rounds, token_rounds, max_len, nbest, prefix, blank_mode, prune_mode,
        eos, merge_mode, quirk, with_lm, late, early;
    double lam;
    unsigned long long hbase, hmod;
};

struct DevState {
    int B, S, K, Tmax, NT, ntile_cols, max_cols, ndx;
    int sk_split;          // CUDA-core GEMMs: K-loop slices per tile (split-K, 1 = off)
    double* sk_scratch;    // [tiles][sk_split][256 x 4 x CJ] fp64 partial tiles
    unsigned* sk_ticket;   // [tiles] arrival tickets (self-resetting)
    int Jp, Hp, Dp;   // bf16 operand row pitches (elements)
    int tc;           // 1 = tensor-core path (bf16 operands staged for TMA)
    int split3;       // 1 = precision fp32 on the tensor cores: every operand row staged as
                      //    three bf16 planes (x = x0 + x1 + x2), plane strides below
    size_t zpl, hpl;  // elements between the planes of z16 / of hA16 and hB16
    int trace;        // measurement aids baked into the plan: 1 = phase trace, 2 = launch timeline
    int probe_on;     // AES++ prefix probes: the joint epilogue also emits, per row, the
                      // logits of the other slots' last tokens (probe[S][K])
    float* probe;
    int round_in_proj;  // 1: the LSTM projection GEMM closes the round (round counter, WHILE
                        //    condition); 0: the select kernel's last CTA does
    // per stream
    int* T;
    int* t;
    int* r;
    int* done;
    int* steps;
    int* col;                 // [B] rounds run by the stream = its next trie column
    unsigned long long* ctr;  // [B, 5]
    // per slot
    double* score;
    int* len;
    unsigned long long* hash;
    int* last;
    int* f;
    int* tnode;
    int* lm_state;
    unsigned char* donated;
    unsigned char* sdonated;
    // prediction-network state pool: P = 2K entries per stream, row b*P + e.
    // A slot points at an entry (pid); blank children share their parent's,
    // token children get a free one -- nothing is copied per round.
    int P;
    int* pid;     // [S]
    int* win;     // [B*P][n]
    float* h;     // [B*P][H]
    float* c;     // [B*P][H]
    float* pred;  // [B*P][J]
    // token rows of the round (LSTM step): pool rows of parent / child, token
    int* upd_src;  // [2][S]
    int* upd_dst;  // [2][S]
    int* upd_tok;  // [2][S]
    // compacted lists [2][S] + counts [2]
    int* act_list;
    int* act_count;
    int* upd_list;
    int* upd_count;
    // joint partials
    // packed record per (slot, partial tile), 16-B aligned, written with
    // vector stores: {max, sum-exp, -, -} then K x {raw, idx, logit, lm}
    float* part;       // [S, NT, 4 + 4K]
    float* blank_logit;// [S]
    float* dur_logit;  // [S, ndx]
    // token trie
    int* st_tok;       // [max_cols, S]
    int* st_prev;      // [max_cols, S]
    signed char* st_dur;  // [max_cols, S]
    int* st_frame;     // [max_cols, B]
    // encoder projection [B, Tmax, J] fp32
    float* encp;
    // inputs, indirect so one captured graph serves any device buffers:
    const float* const* enc_pp;  // -> enc [B, Tmax, D] fp32
    const int* const* len_pp;    // -> lengths [B]
    // tensor-core operands, bf16, compacted rows
    __nv_bfloat16* z16;    // [S, Jp] joint input of the next round, row = act_pos
    __nv_bfloat16* hA16;   // [S, Hp] parent h of token rows, row = upd_pos
    __nv_bfloat16* hB16;   // [S, Hp] new h of token rows, row = upd_pos
    __nv_bfloat16* enc16;  // [B*Tmax, Dp] encoder frames
    int* act_pos;          // [S] row of the slot in next round's active list or -1
    int* upd_pos;          // [S] row of the slot in this round's token list or -1
    // loop control
    int* g;           // rounds executed (statistics)
    int* live;        // this round had a decoding stream (set by the joint; unrolled WHILE
                      // bodies run a few no-op rounds at the end of a decode)
    int* n_done;      // finished streams
    int* sel_blocks;  // select CTAs finished this round (last-block bookkeeping)
    // outputs
    int* out_count;    // [B]
    int* out_len;      // [B, nbest]
    double* out_score; // [B, nbest]
    int* out_tok;      // [B, nbest, max_len]
    int* out_frame;
    int* out_dur;
};

}  // namespace tbeam_dev
