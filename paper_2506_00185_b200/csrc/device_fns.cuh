// Device restatements of the reference's scalar helpers.
//   update_hash      hyp_store.cpp:13-37   (Mersenne-61 fast path + generic modulus)
//   logadd           hyp_store.cpp:39-44
//   log1mexp         fusion.cpp:11-22
//   LM queries       ngram_lm.cpp:320-438  (find_child, score_internal,
//                    score_token, score_eos, score_vocab value, advance)
#pragma once

#include <cmath>
#include <cstdint>

#include "engine.cuh"

namespace tbeam_dev {

__device__ __forceinline__ unsigned long long d_update_hash(unsigned long long h, int tok,
                                                            unsigned long long base,
                                                            unsigned long long mod) {
    const unsigned __int128 x = static_cast<unsigned __int128>(h) * base +
                                static_cast<unsigned long long>(tok) + 1ull;
    if (mod == kMersenne61) {
        unsigned long long r = static_cast<unsigned long long>(x & kMersenne61) +
                               static_cast<unsigned long long>(x >> 61);
        r = (r & kMersenne61) + (r >> 61);
        if (r >= kMersenne61) r -= kMersenne61;
        return r;
    }
    return static_cast<unsigned long long>(x % mod);
}

__device__ __forceinline__ double d_logadd(double a, double b) {
    if (a == -INFINITY) return b;
    if (b == -INFINITY) return a;
    const double m = fmax(a, b);
    return m + log1p(exp(fmin(a, b) - m));
}

__device__ __forceinline__ double d_merge(double a, double b, int merge_mode) {
    return merge_mode == 1 ? fmax(a, b) : d_logadd(a, b);
}

// (out of line: one copy of the fp64 log1p/expm1 code serves every call site)
static __device__ __noinline__ double d_log1mexp(double x) {
    if (x >= 0.0) return -INFINITY;  // x == 0 (x > 0 cannot occur for a log-prob)
    if (x > -0.69314718055994530942) return log(-expm1(x));
    return log1p(-exp(x));
}

// ---- n-gram LM --------------------------------------------------------------

__device__ __forceinline__ int lm_find_child(const DevLm& lm, int node, int tok) {
    if (node == 0) return tok >= 0 && tok < lm.n_root ? lm.root[tok] : -1;  // dense root level
    int lo = lm.cbeg[node], hi = lm.cend[node];
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (lm.etok[mid] < tok) lo = mid + 1;
        else hi = mid;
    }
    if (lo < lm.cend[node] && lm.etok[lo] == tok) return lm.enode[lo];
    return -1;
}

static __device__ __noinline__ double lm_score_internal(const DevLm& lm, int state, int tok) {
    double acc = 0.0;
    int c = state;
    while (true) {
        const int node = lm_find_child(lm, c, tok);
        if (node >= 0 && !isnan(lm.prob[node])) return fmax(acc + lm.prob[node], kLogZeroFloor);
        if (c == 0) return kLogZeroFloor;
        acc += lm.backoff[c];
        c = lm.suffix[c];
    }
}

// NGramLm::score_token (ngram_lm.cpp:346-356)
__device__ __forceinline__ double lm_score_token(const DevLm& lm, int state, int tok) {
    const int it = lm.remap[tok];
    if (it < 0) return kLogZeroFloor;
    return lm_score_internal(lm, state, it);
}

// NGramLm::score_eos (ngram_lm.cpp:358-361)
__device__ __forceinline__ double lm_score_eos(const DevLm& lm, int state) {
    return lm_score_internal(lm, state, lm.V + 1);
}

// One entry of NGramLm::score_vocab's row (ngram_lm.cpp:363-416): deepest
// level holding the token with a probability, else <unk> under the whole
// backoff chain, else the floor.
static __device__ __noinline__ double lm_vocab_value(const DevLm& lm, int state, int tok) {
    double acc = 0.0;
    int c = state;
    while (true) {
        const int node = lm_find_child(lm, c, tok);
        if (node >= 0 && !isnan(lm.prob[node])) return fmax(acc + lm.prob[node], kLogZeroFloor);
        if (c == 0) break;
        acc += lm.backoff[c];
        c = lm.suffix[c];
    }
    return isfinite(lm.unk_prob) ? fmax(acc + lm.unk_prob, kLogZeroFloor) : kLogZeroFloor;
}

// NGramLm::advance (ngram_lm.cpp:418-438)
static __device__ __noinline__ int lm_advance(const DevLm& lm, int state, int tok) {
    const int it = lm.remap[tok];
    if (it < 0) return 0;
    int c = state;
    while (true) {
        const int node = lm_find_child(lm, c, it);
        if (node >= 0) return lm.depth[node] == lm.order ? lm.suffix[node] : node;
        if (c == 0) return 0;
        c = lm.suffix[c];
    }
}

// Fused selection value of a token column (decoder.cpp:47-61 / fusion.cpp:24-43)
// from its logit, the row normaliser and (late) its LM value.
__device__ __forceinline__ double fused_token(const DevCfg& cfg, double logit, double lse,
                                              double lmv, double l1m_blank) {
    const double asr = logit - lse;
    if (!cfg.late) return asr;
    if (cfg.blank_mode == 0) return asr + cfg.lam * lmv;
    return asr + cfg.lam * (lmv + l1m_blank);
}

__device__ __forceinline__ double fused_blank(const DevCfg& cfg, double asr_blank) {
    if (cfg.with_lm && cfg.blank_mode == 1) return (1.0 + cfg.lam) * asr_blank;
    return asr_blank;
}

// out-of-line fp64 exp / log for the latency-bound per-round kernels (their
// code is fetched cold each round: one copy instead of one per call site)
#ifndef TBEAM_MATH_CALL  // inline: measured 0.15 us/round faster select
static __device__ __forceinline__ double d_exp(double x) { return exp(x); }
static __device__ __forceinline__ double d_log(double x) { return log(x); }
#else
static __device__ __noinline__ double d_exp(double x) { return exp(x); }
static __device__ __noinline__ double d_log(double x) { return log(x); }
#endif

__device__ __forceinline__ float bf16_round(float x) {
    return __bfloat162float(__float2bfloat16_rn(x));
}

// Tensor-core operand stores.  bf16 precision: one plane, bf16(x).  fp32
// precision on the tensor cores (split = st.split3): three planes
// x0 = bf16(x), x1 = bf16(x - x0), x2 = bf16(x - x0 - x1) -- each remainder is
// exact in fp32 and x2 takes the last <= 8 significant bits, so
// x = x0 + x1 + x2 exactly; `plane` = elements between planes.
__device__ __forceinline__ void put_op(__nv_bfloat16* dst, size_t plane, int split, float x) {
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    dst[0] = h;
    if (split) {
        x -= __bfloat162float(h);
        const __nv_bfloat16 h1 = __float2bfloat16_rn(x);
        dst[plane] = h1;
        dst[2 * plane] = __float2bfloat16_rn(x - __bfloat162float(h1));
    }
}
__device__ __forceinline__ uint32_t pack_bf16x2(float& a, float& b) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    a -= __low2float(h);
    b -= __high2float(h);
    return *reinterpret_cast<const uint32_t*>(&h);
}
// 4 consecutive elements (8-byte aligned destination)
__device__ __forceinline__ void put_op4(__nv_bfloat16* dst, size_t plane, int split, float a, float b, float c,
                                        float d) {
    uint2 pk;
    pk.x = pack_bf16x2(a, b);
    pk.y = pack_bf16x2(c, d);
    *reinterpret_cast<uint2*>(dst) = pk;
    if (split) {
#pragma unroll
        for (int p = 1; p < 3; ++p) {
            pk.x = pack_bf16x2(a, b);
            pk.y = pack_bf16x2(c, d);
            *reinterpret_cast<uint2*>(dst + p * plane) = pk;
        }
    }
}

}  // namespace tbeam_dev
