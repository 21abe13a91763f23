// Search-side kernels of the decode loop, sm_100a.
//
// select_kernel: one CTA per stream does everything BeamEngine::run_lane does
// between two model calls (decoder.cpp:160-324), on device:
//   combine the joint's per-tile partials -> row log-softmax normaliser, blank
//   and (TDT) duration log-probs, per-row top-K fused tokens;
//   AES++ maximum-length prefix pass (decoder.cpp:186-229);
//   candidate formation (decoder.cpp:231-254) incl. carries of complete slots;
//   blank-column recombination by HypKey (decoder.cpp:256-277);
//   prune_topk total order (hyp_store.cpp:199-228);
//   expansion + token-trie append + hash/length/last update + LM advance and
//   early-pruning LM term (decoder.cpp:282-324, hyp_store.cpp:89-135);
//   per-stream frame/round state machine (decoder.cpp:143-158) and counters;
//   the compacted active-row list of the next round.
// pred_update: prediction-network state of the new beam, gathered by parent
// (window shift, decoder.cpp:288-318 / model.cpp:109-121; LSTM copy).
// control: advances the round counter and sets the CUDA-graph WHILE condition.
// finalize: EOS term, ranking and n-best backtrace (decoder.cpp:329-355,
// hyp_store.cpp:151-167) with alignments.
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstdint>

#include "device_fns.cuh"
#include "engine.cuh"
#include "kernels.h"
#include "tc_common.cuh"

#ifndef TBEAM_EXACT_EXP
#define TBEAM_EXACT_EXP 0
#endif

namespace tbeam_dev {

namespace {

// bytes of a combine warp's data area: the staged joint partials, reused
// after the merge as the TDT (token, duration) combo scratch and (warp 0) the
// pruned-rank scratch -- sized to the largest, no fixed minimum: at the bench
// shape the select CTA then fits on an SM beside a resident joint CTA (whose
// 207 KB smem would otherwise delay the select's launch to the joint's exit)
__host__ __device__ inline size_t stg_data_bytes(int K, int ndx, size_t nstage_floats) {
    size_t b = 4 * nstage_floats;
    const size_t tdt = ndx > 1 ? 16 * static_cast<size_t>(K) * ndx : 0;
    const size_t prune = K * (K + ndx) > 32 ? 128 * 20 : 0;
    b = b > tdt ? b : tdt;
    b = b > prune ? b : prune;
    return (b + 15) / 16 * 16;
}

struct SelSmem {
    // byte offsets of every array in the dynamic shared buffer
    size_t sc, lse, asrb, fbl, l1m, dlp, tkv, csc, nsc, edon, cidx, hs, ln, ls, fr, tn, lmst,
        act, tkn, tki, tkw, ck, cdi, cdest, sel, ea, ec, don, stg, total;
    int cw;         // warps that combine joint partials (each stages one slot's records)
    size_t stg_per; // bytes of one warp's staging area
    // nstage = per-warp staging floats (NT records of the joint partials), nw = warps
    __host__ __device__ SelSmem(int K, int ndx, int nstage = 0, int nw = 0) {
        const int RS = K + ndx;
        size_t o = 0;
        auto take = [&](size_t bytes) {
            const size_t at = o;
            o += (bytes + 15) & ~size_t(15);
            return at;
        };
        sc = take(8 * K);
        lse = take(8 * K);
        asrb = take(8 * K);
        fbl = take(8 * K);
        l1m = take(8 * K);
        dlp = take(8 * K * ndx);
        tkv = take(8 * K * K);
        csc = take(8 * K * RS);
        nsc = take(8 * K * ndx);
        edon = take(8 * K * K);
        cidx = take(8 * K * RS);
        hs = take(8 * K);
        ln = take(4 * K);
        ls = take(4 * K);
        fr = take(4 * K);
        tn = take(4 * K);
        lmst = take(4 * K);
        act = take(4 * K);
        tkn = take(4 * K);
        tki = take(4 * K * K);
        ck = take(4 * K * RS);
        cdi = take(4 * K * RS);
        cdest = take(4 * K * RS);
        sel = take(4 * K);
        ea = take(4 * K * K);
        ec = take(4 * K * K);
        don = take(4 * K);
        tkw = take(4 * K * K);
        // per warp: staging of the joint partials (also the TDT combo
        // scratch, >= 4 KB) + NT list heads; as many warps as 144 KB holds
        const size_t per = stg_data_bytes(K, ndx, static_cast<size_t>(nstage)) +
                           (4 * static_cast<size_t>(nstage / 8 + 1) + 15) / 16 * 16;
        stg_per = per;
        cw = nw;
        while (cw > 1 && per * cw > 144 * 1024) --cw;
        stg = take(per * cw);
        total = o;
    }
};

#ifdef TBEAM_OLD_DUR
#define TDUR(d) m.durations[d]
#else
#define TDUR(d) s_dur[warp][d]
#endif
// cold-path hint: the select runs once per round with its code fetched cold,
// so rarely-taken blocks (traces, AES prefix pass, finished streams) are laid
// out of line and the common path stays sequential in the instruction stream
#ifdef TBEAM_NO_EXPECT
#define TB_UNLIKELY(x) (x)
#else
#define TB_UNLIKELY(x) __builtin_expect(!!(x), 0)
#endif
// measurement switches (variants built with -D, selected with TBEAM_LIB)
#ifndef TBEAM_STAGE_BATCH
#define TBEAM_STAGE_BATCH 4
#endif
#ifdef TBEAM_MERGE_CALL
#define TBEAM_MERGE_ATTR __noinline__
#else
#define TBEAM_MERGE_ATTR __forceinline__  // measured 0.2 us/round faster than a call
#endif

__device__ __forceinline__ bool beats_f(float va, int ia, float vb, int ib) {
    return (va > vb) | ((va == vb) & (ia < ib));
}

// Compact (non-inlined, loop-based) warp helpers for the select kernel: the
// decode loop runs each kernel once per round, so the select's executed code
// is fetched cold every round -- code size, not arithmetic, sets its latency.

// Top-K (value desc, key asc) of n <= 2048 smem entries by one warp; entry e
// is position idx[e] (idx == nullptr: e itself) of val/key; -inf entries are
// not candidates.  out[j] = entry of the j-th winner; returns the count.
__device__ __noinline__ int warp_topk_smem(const double* val, const long long* key, const int* idx, int n, int K,
                                           int* out) {
    const int lane = threadIdx.x & 31;
    unsigned long long taken = 0ull;  // bit u: entry lane + 32u consumed
    int found = 0;
    for (int j = 0; j < K; ++j) {
        double bv = -INFINITY;
        long long bk = 0x7fffffffffffffffll;
        int be = -1;
#pragma unroll 1
        for (int e = lane, u = 0; e < n; e += 32, ++u) {
            if ((taken >> u) & 1ull) continue;
            const int y = idx ? idx[e] : e;
            const double v = val[y];
            if (v == -INFINITY) continue;
            const long long k = key[y];
            if (v > bv || (v == bv && k < bk)) {
                bv = v;
                bk = k;
                be = e;
            }
        }
        double wv = bv;
        long long wk = bk;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, wv, o);
            const long long ok = __shfl_xor_sync(0xffffffffu, wk, o);
            if (ov > wv || (ov == wv && ok < wk)) {
                wv = ov;
                wk = ok;
            }
        }
        if (wv == -INFINITY) break;
        if (be >= 0 && bk == wk) {  // keys are unique: exactly one owner
            out[j] = be;
            taken |= 1ull << ((be - lane) >> 5);
        }
        ++found;
    }
    __syncwarp();
    return found;
}

// The same for n <= 32 * U in one pass: lane l owns entries l + 32u and
// counts the entries that beat each of them (a broadcast smem loop, no
// shuffle chains); the winners write out[rank] = entry.
template <int U>
__device__ __forceinline__ int warp_rank(const double* val, const long long* key, int n, int K, int* out) {
    const int lane = threadIdx.x & 31;
    double v[U];
    long long k[U];
    int rank[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int e = lane + 32 * u;
        v[u] = e < n ? val[e] : -INFINITY;
        k[u] = e < n ? key[e] : 0;
        rank[u] = 0;
    }
    // (non-short-circuit & / |: predicated compares, no per-lane branches; a
    // -inf or NaN entry never beats a valid one, so it needs no test)
#pragma unroll 4
    for (int e = 0; e < n; ++e) {
        const double ve = val[e];
        const long long ke = key[e];
#pragma unroll
        for (int u = 0; u < U; ++u)
            rank[u] += static_cast<int>((ve > v[u]) | ((ve == v[u]) & (ke < k[u])));
    }
    int nv = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const bool valid = v[u] > -INFINITY;  // (a NaN is never a candidate, as in warp_topk_smem)
        if (valid && rank[u] < K) out[rank[u]] = lane + 32 * u;
        nv += __popc(__ballot_sync(0xffffffffu, valid));
    }
    __syncwarp();
#ifdef TBEAM_RANK_CHECK
    {
        const int f = nv < K ? nv : K;
        bool bad = false;
        if (lane == 0)
            for (int q = 0; q < f; ++q) {
                const int e = out[q];
                if (e < 0 || e >= n || !(val[e] > -INFINITY)) bad = true;
                for (int q2 = 0; q2 < q; ++q2) if (out[q2] == e) bad = true;
            }
        if (lane == 0 && bad) {
            printf("RANKBAD blk %d warp %d n %d K %d nv %d\n", blockIdx.x, threadIdx.x >> 5, n, K, nv);
            for (int e = 0; e < n; ++e) printf("  e %d v %.17g k %lld\n", e, val[e], key[e]);
            for (int q = 0; q < f; ++q) printf("  out %d = %d\n", q, out[q]);
        }
        __syncwarp();
    }
#endif
    return nv < K ? nv : K;
}
// top-K of n smem entries by one warp: counting ranks up to 128 entries,
// else K rounds of warp arg-max
// NMAX: a compile-time bound on n (0 = none) -- only the variants it admits
// are compiled into the caller
template <int NMAX>
__device__ __forceinline__ int warp_select(const double* val, const long long* key, int n, int K, int* out) {
#ifdef TBEAM_OLD_SELECT
    return warp_topk_smem(val, key, nullptr, n, K, out);
#endif
    constexpr bool b32 = NMAX == 0 || NMAX > 32, b64 = NMAX == 0 || NMAX > 64, b128 = NMAX == 0 || NMAX > 128;
    if (!b32 || n <= 32) return warp_rank<1>(val, key, n, K, out);
    if constexpr (b32) {
        if (!b64 || n <= 64) return warp_rank<2>(val, key, n, K, out);
        if constexpr (b64) {
            if (!b128 || n <= 128) return warp_rank<4>(val, key, n, K, out);
            if constexpr (b128) return warp_topk_smem(val, key, nullptr, n, K, out);
        }
    }
    return 0;
}

// prune_topk over the candidate regions (slot i: entries [i*RS, (i+1)*RS),
// its K token entries first, non-increasing): a slot whose K-th token entry
// is valid has K entries at least that large, so the largest such value over
// the slots bounds the global K-th best from below; only entries reaching it
// (compacted into scratch) go through the counting rank.  Falls back to warp
// arg-max rounds when more than 128 entries survive.
__device__ __forceinline__ int warp_pruned_rank(const double* val, const long long* key, int n, int K, int RS,
                                                int* out, unsigned char* scratch) {
    const int lane = threadIdx.x & 31;
    double th = lane < K ? val[lane * RS + K - 1] : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) th = fmax(th, __shfl_xor_sync(0xffffffffu, th, o));
    double* sv = reinterpret_cast<double*>(scratch);
    long long* sk = reinterpret_cast<long long*>(scratch + 128 * 8);
    int* si = reinterpret_cast<int*>(scratch + 128 * 16);
    int m = 0;
    #pragma unroll 1
    for (int e0 = 0; e0 < n; e0 += 32) {
        const int e = e0 + lane;
        const double v = e < n ? val[e] : -INFINITY;
        const bool keep = (v > -INFINITY) & (v >= th);
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        const int pos = m + __popc(bal & ((1u << lane) - 1u));
        if (keep && pos < 128) {
            sv[pos] = v;
            sk[pos] = key[e];
            si[pos] = e;
        }
        m += __popc(bal);
    }
    __syncwarp();
    if (m > 128) return warp_topk_smem(val, key, nullptr, n, K, out);
    const int f = m <= 32 ? warp_rank<1>(sv, sk, m, K, out) : m <= 64 ? warp_rank<2>(sv, sk, m, K, out)
                                                                 : warp_rank<4>(sv, sk, m, K, out);
    const int x = lane < f ? si[out[lane]] : 0;
    __syncwarp();
    if (lane < f) out[lane] = x;
    __syncwarp();
    return f;
}

// Register top-KM of NT sorted lists (KM <= 16, K <= KM): each lane merges
// its own lists (q = lane + 32u) into one sorted KM-list, then five butterfly
// steps merge the lanes' lists -- a bitonic merge of two sorted lists keeps
// the better half (max(A[q], B[KM-1-q])) and a log2(KM)-stage bitonic sort
// restores the order; all indices static.  Order: raw desc, column asc.
// Then lane j (< found) holds nothing special: every lane ends with the same
// list; tki/lg/lmv are written by lane 0 reading the winners' records.
template <int KM>
__device__ __forceinline__ bool bt_better(float av, int ai, float bv, int bi) {
    return (av > bv) | ((av == bv) & (ai < bi));
}
template <int KM>
__device__ __forceinline__ void bt_sort(float (&v)[KM], int (&ix)[KM], int (&org)[KM]) {
    // bitonic sequence -> sorted (desc): stages of compare-exchange at distance d
#pragma unroll
    for (int d = KM / 2; d >= 1; d >>= 1)
#pragma unroll
        for (int q = 0; q < KM; ++q)
            if ((q & d) == 0 && !bt_better<KM>(v[q], ix[q], v[q + d], ix[q + d])) {
                const float tv = v[q];
                const int ti = ix[q], to = org[q];
                v[q] = v[q + d];
                ix[q] = ix[q + d];
                org[q] = org[q + d];
                v[q + d] = tv;
                ix[q + d] = ti;
                org[q + d] = to;
            }
}
template <int KM>
__device__ __forceinline__ void bt_merge(float (&v)[KM], int (&ix)[KM], int (&org)[KM], const float (&bv)[KM],
                                         const int (&bi)[KM], const int (&bo)[KM]) {
#pragma unroll
    for (int q = 0; q < KM; ++q)
        if (!bt_better<KM>(v[q], ix[q], bv[KM - 1 - q], bi[KM - 1 - q])) {
            v[q] = bv[KM - 1 - q];
            ix[q] = bi[KM - 1 - q];
            org[q] = bo[KM - 1 - q];
        }
    bt_sort<KM>(v, ix, org);
}
template <int KM>
__device__ TBEAM_MERGE_ATTR int warp_merge_reg(const float* w, int NT, int ps, int K, int* tki, double* lg, double* lmv) {
    const int lane = threadIdx.x & 31;
    float v[KM];
    int ix[KM], org[KM];
#pragma unroll
    for (int q = 0; q < KM; ++q) {
        v[q] = -INFINITY;
        ix[q] = 0x7fffffff;
        org[q] = -1;
    }
    #pragma unroll 1
    for (int l = lane; l < NT; l += 32) {  // this lane's lists, each sorted
        float bv[KM];
        int bi[KM], bo[KM];
#pragma unroll
        for (int q = 0; q < KM; ++q) {
            bv[q] = -INFINITY;
            bi[q] = 0x7fffffff;
            bo[q] = -1;
            if (q < K) {
                const float2 e = *reinterpret_cast<const float2*>(w + l * ps + 4 + 4 * q);
                if (__float_as_int(e.y) >= 0) {
                    bv[q] = e.x;
                    bi[q] = __float_as_int(e.y);
                    bo[q] = l * ps + 4 + 4 * q;
                }
            }
        }
        bt_merge<KM>(v, ix, org, bv, bi, bo);
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        float bv[KM];
        int bi[KM], bo[KM];
#pragma unroll
        for (int q = 0; q < KM; ++q) {
            bv[q] = __shfl_xor_sync(0xffffffffu, v[q], o);
            bi[q] = __shfl_xor_sync(0xffffffffu, ix[q], o);
            bo[q] = __shfl_xor_sync(0xffffffffu, org[q], o);
        }
        bt_merge<KM>(v, ix, org, bv, bi, bo);
    }
    int found = 0;
#pragma unroll
    for (int q = 0; q < KM; ++q) found += (q < K && ix[q] != 0x7fffffff) ? 1 : 0;
    // lane j publishes winner j (static selects, no dynamic register index)
    int myo = -1, myi = 0;
#pragma unroll
    for (int q = 0; q < KM; ++q)
        if (q == lane) {
            myo = org[q];
            myi = ix[q];
        }
    if (lane < found) {
        const float2 l2 = *reinterpret_cast<const float2*>(w + myo + 2);
        tki[lane] = myi;
        lg[lane] = static_cast<double>(l2.x);
        lmv[lane] = static_cast<double>(l2.y);
    }
    __syncwarp();
    return found;
}

// K-way merge of NT lists staged at w (list q: K float4 records from
// w[q*ps + 4], sorted by raw desc / idx asc; idx < 0 = empty) into the top-K
// columns: tki[j] = column, lg[j] / lmv[j] = its logit / LM value.  heads:
// per-warp scratch of NT ints.  Returns the count.
__device__ __noinline__ int warp_merge_lists(const float* w, int NT, int ps, int K, int* heads, int* tki, double* lg,
                                             double* lmv) {
    // lane l owns lists l + 32u (NT <= 256: u < 8) and keeps each one's head
    // record (value, column) in registers: a pick is a register arg-max per
    // lane + a warp arg-max; only the winner's list advances (one smem load)
    (void)heads;
    constexpr int UM = 8;
    const int lane = threadIdx.x & 31;
    float hv[UM];
    int hc[UM], hp[UM] = {};
    auto load_head = [&](int u) {
        const int q = lane + 32 * u;
        float v = -INFINITY;
        int c = 0x7fffffff;
        if (q < NT && hp[u] < K) {
            const float2 e = *reinterpret_cast<const float2*>(w + q * ps + 4 + 4 * hp[u]);
            const int ix = __float_as_int(e.y);
            v = ix >= 0 ? e.x : -INFINITY;
            c = ix >= 0 ? ix : 0x7fffffff;
        }
        hv[u] = v;
        hc[u] = c;
    };
#pragma unroll
    for (int u = 0; u < UM; ++u) {
        hp[u] = 0;
        load_head(u);
    }
    int found = 0;
    #pragma unroll 1
    for (int j = 0; j < K; ++j) {
        float bv = -INFINITY;
        int bi = 0x7fffffff, bu = -1;
#pragma unroll
        for (int u = 0; u < UM; ++u) {
            const bool b = (hc[u] != 0x7fffffff) & beats_f(hv[u], hc[u], bv, bi);
            bv = b ? hv[u] : bv;
            bi = b ? hc[u] : bi;
            bu = b ? u : bu;
        }
        float wv = bv;
        int wi = bi;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, wv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, wi, o);
            const bool b = beats_f(ov, oi, wv, wi);
            wv = b ? ov : wv;
            wi = b ? oi : wi;
        }
        if (wi == 0x7fffffff) break;
        if (bu >= 0 && bi == wi) {  // column ids are unique: exactly one owner
#pragma unroll
            for (int u = 0; u < UM; ++u)
                if (u == bu) {
                    const int q = lane + 32 * u;
                    const float2 l = *reinterpret_cast<const float2*>(w + q * ps + 4 + 4 * hp[u] + 2);
                    tki[j] = wi;
                    lg[j] = static_cast<double>(l.x);
                    lmv[j] = static_cast<double>(l.y);
                    hp[u] += 1;
                    load_head(u);
                }
        }
        ++found;
    }
    __syncwarp();
    return found;
}


}  // namespace

// 4 warps: one slot per warp (more slots loop); small CTAs keep many streams resident
int select_threads(int K) {
    if (const char* e = std::getenv("TBEAM_SEL_THREADS")) {  // measurement override
        const int v = std::atoi(e);
        if (v == 128 || v == 256) return v;
    }
    // one warp per slot in the combine up to 8 slots (K >= 8: measured
    // 11 us/round faster at K = 8); K = 4 too since round 2 (the staging and
    // pool phases use the extra warps: select 11.9 -> 10.6 us busy, round
    // 34.4 -> 32.9 us at the bench shape)
    return K >= 4 ? 256 : 128;
}
size_t select_smem_bytes(int K, int ND, int NT) {
    return SelSmem(K, ND > 0 ? ND : 1, NT * part_stride(K), select_threads(K) / 32).total;
}

// phase trace of every select CTA (SM clock), measurement aid: per-CTA
// accumulators [1024 CTAs][8] (phases 1..5, 6 = tail after the stream work,
// 7 = the stream work, 0 = launches); thread 0 keeps marks in shared memory
// and flushes once at the end, so tracing stays off the critical path
#ifndef TBEAM_DONOR_UNROLL
#define TBEAM_DONOR_UNROLL 20  // (4: C5 donor values 14.0k -> 10.9k cycles per select CTA-round with 20)
#endif
constexpr int kDonorUnroll = TBEAM_DONOR_UNROLL;  // AES++ donor dot products: loads in flight per batch
constexpr int kSelTraceCtas = 1024;
constexpr int kSelTr = 32;  // trace slots per CTA
__device__ long long g_sel_trace[kSelTraceCtas * kSelTr];
__shared__ long long s_sel_tr[kSelTr];
// device-wide launch timeline (tc_common.cuh), kernel slot 3 = select
__device__ unsigned long long g_tl_sel[kTlRounds * 4 * 4];
// sub-phase marks inside the combine (warp 0, slot 0), slots 8..15
#define SUB_MARK(k)                                                                      \
    do {                                                                                 \
        if (TB_UNLIKELY((st.trace & 1) && threadIdx.x == 0 && i == 0)) {                \
            const long long _t = clock64();                                              \
            s_sel_tr[k] += _t - sub_t0;                                                  \
            sub_t0 = _t;                                                                 \
        }                                                                                \
    } while (0)
#define SEL_MARK(k)                                                                      \
    do {                                                                                 \
        if (TB_UNLIKELY((st.trace & 1) && threadIdx.x == 0)) {                           \
            const long long _t = clock64();                                              \
            s_sel_tr[k] += _t - sel_t0;                                                  \
            sel_t0 = _t;                                                                 \
        }                                                                                \
    } while (0)

// ---------------------------------------------------------------------------
// init: fresh store (hyp_store.cpp:46-67) + start prediction state
// grid B, block 128
// ---------------------------------------------------------------------------
__global__ void init_kernel(DevModel m, DevLm lm, DevCfg cfg, DevState st) {
    const int b = blockIdx.x;
    const int K = cfg.K;
    if (threadIdx.x < K) {
        const int i = threadIdx.x;
        const int s = b * K + i;
        st.score[s] = i == 0 ? 0.0 : -INFINITY;
        st.len[s] = 0;
        st.hash[s] = 0ull;
        st.last[s] = -1;
        st.f[s] = 0;
        st.tnode[s] = -1;
        st.lm_state[s] = lm.present ? lm.initial : 0;
        st.sdonated[s] = 0;
        st.pid[s] = 0;
        if (st.tc) {
            st.act_pos[s] = i == 0 ? b : -1;
            st.upd_pos[s] = -1;
        }
    }
    if (threadIdx.x == 0) {
        st.T[b] = (*st.len_pp)[b];
        st.t[b] = 0;
        st.r[b] = 0;
        st.done[b] = 0;
        st.steps[b] = 0;
        st.col[b] = 0;
        for (int q = 0; q < 5; ++q) st.ctr[b * 5 + q] = 0ull;
        st.act_list[b] = b * K;  // parity 0 list: slot 0 of every stream
        if (b == 0) {
            st.act_count[0] = st.B;
            st.act_count[1] = 0;
            st.upd_count[0] = 0;
            st.upd_count[1] = 0;
            *st.g = 0;
            *st.live = 1;
            *st.n_done = 0;
            *st.sel_blocks = 0;
        }
    }
    // prediction-state pool: entry 0 of the stream = start state, every slot -> 0
    {
        const size_t row = static_cast<size_t>(b) * st.P;
        if (m.pred_kind == 1) {
            for (int u = threadIdx.x; u < m.H; u += blockDim.x) {
                st.h[row * m.H + u] = m.h0[u];
                st.c[row * m.H + u] = m.c0[u];
            }
            for (int j = threadIdx.x; j < m.J; j += blockDim.x) st.pred[row * m.J + j] = m.pred0[j];
        } else {
            const float inv = m.n > 0 ? 1.0f / m.n : 0.f;
            for (int j = threadIdx.x; j < m.J; j += blockDim.x) {
                float acc = 0.f;
                for (int q = 0; q < m.n; ++q) acc += inv * m.table[static_cast<size_t>(m.V) * m.J + j];
                st.pred[row * m.J + j] = m.b_pred[j] + acc;
            }
            if (threadIdx.x == 0)
                for (int q = 0; q < m.n; ++q) st.win[row * m.n + q] = -1;
        }
    }
    __syncthreads();
    if (st.tc) {
        // first round's joint operand: slot 0 of stream b at frame 0 -> row b
        __syncthreads();
        const float* ep = st.encp + static_cast<size_t>(b) * st.Tmax * m.J;
        const float* pp = st.pred + static_cast<size_t>(b) * st.P * m.J;
        for (int j = threadIdx.x; j < m.J; j += blockDim.x)
            put_op(st.z16 + static_cast<size_t>(b) * st.Jp + j, st.zpl, st.split3, tanhf(ep[j] + pp[j]));
    }
}

// fp32 encoder frames -> bf16 TMA operand rows
__global__ void enc_to_bf16_kernel(DevModel m, DevState st, int rows) {
    const float* enc = *st.enc_pp;
    const size_t n = static_cast<size_t>(rows) * m.D;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t r = i / m.D, d = i % m.D;
        st.enc16[r * st.Dp + d] = __float2bfloat16_rn(enc[i]);
    }
}

// ---------------------------------------------------------------------------
// select: one CTA per stream, warp-centric.  Warp w owns slots w, w+NW, ...:
// it stages the slot's joint partials, reduces them (row normaliser, blank /
// duration log-probs, top-K fused tokens) and writes the slot's candidate
// region.  After one barrier, warps recombine the frame-leaving blank column,
// warp 0 ranks (prune_topk's order), expands the beam, runs the stream's
// frame/round state machine and publishes the next round's rows; after a
// second barrier every warp stages the prediction-network operands.  Global
// loads of a phase are issued together, counters live in shared memory.
// ---------------------------------------------------------------------------
// LSTM / TDT / LM: compile-time switches (dead paths vanish from the code the
// kernel fetches every round)
template <bool LSTM, bool TDT, bool LM, int KT>
__device__ __forceinline__ void select_stream(const DevModel& m, const DevLm& lm, const DevCfg& cfg,
                                           const DevState& st, const SelSmem& L, const int par, const int col,
                                           const int t, const int r, const int T, const int dn) {
    const int b = blockIdx.x;
    extern __shared__ __align__(16) unsigned char smem[];
    // KT: the beam width when the kernel is specialised for it (1, 8, 16),
    // else 0 and K comes from the config -- compile-time K folds the slot
    // loops, the candidate-region divisions and the merge / rank dispatch
    const int K = KT > 0 ? KT : cfg.K, V = m.V, R = m.R, ND = TDT ? m.ND : 0, ndx = TDT ? st.ndx : 1, RS = K + ndx;
    constexpr int NPRE = KT > 0 ? KT * kMaxDur : 0;                     // bound on a slot's TDT combos
    double* sc = reinterpret_cast<double*>(smem + L.sc);
    double* lse = reinterpret_cast<double*>(smem + L.lse);
    double* asrb = reinterpret_cast<double*>(smem + L.asrb);
    double* fbl = reinterpret_cast<double*>(smem + L.fbl);
    double* l1m = reinterpret_cast<double*>(smem + L.l1m);
    double* dlp = reinterpret_cast<double*>(smem + L.dlp);
    double* tkv = reinterpret_cast<double*>(smem + L.tkv);
    double* csc = reinterpret_cast<double*>(smem + L.csc);
    double* nsc = reinterpret_cast<double*>(smem + L.nsc);
    double* edon = reinterpret_cast<double*>(smem + L.edon);
    long long* cidx = reinterpret_cast<long long*>(smem + L.cidx);
    unsigned long long* hs = reinterpret_cast<unsigned long long*>(smem + L.hs);
    int* ln = reinterpret_cast<int*>(smem + L.ln);
    int* ls = reinterpret_cast<int*>(smem + L.ls);
    int* fr = reinterpret_cast<int*>(smem + L.fr);
    int* tn = reinterpret_cast<int*>(smem + L.tn);
    int* lmst = reinterpret_cast<int*>(smem + L.lmst);
    int* act = reinterpret_cast<int*>(smem + L.act);
    int* tkn = reinterpret_cast<int*>(smem + L.tkn);
    int* tki = reinterpret_cast<int*>(smem + L.tki);
    int* ck = reinterpret_cast<int*>(smem + L.ck);
    int* cdi = reinterpret_cast<int*>(smem + L.cdi);
    int* cdest = reinterpret_cast<int*>(smem + L.cdest);
    int* sel = reinterpret_cast<int*>(smem + L.sel);
    int* ea = reinterpret_cast<int*>(smem + L.ea);
    int* ec = reinterpret_cast<int*>(smem + L.ec);
    int* don = reinterpret_cast<int*>(smem + L.don);
    int* pick = reinterpret_cast<int*>(smem + L.tkw);  // [K][K] TDT combo picks
    float* stg = reinterpret_cast<float*>(smem + L.stg);
    __shared__ int n_edges, n_final, n_early;
    __shared__ int s_par[kMaxBeam], s_tok[kMaxBeam], s_upos[kMaxBeam], s_apos[kMaxBeam];
    __shared__ int s_pid[kMaxBeam], s_npid[kMaxBeam];  // prediction-state pool entries (old / new)
    __shared__ unsigned long long s_ctr[5];
    __shared__ int s_t, s_done;
    __shared__ int s_dur[8][kMaxDur];      // TDT durations, one copy per warp (no divergent param-space loads)
    __shared__ unsigned s_dupm[kMaxBeam];  // recombination: slots with the same (hash, length, last)

    const int tid = threadIdx.x, nthr = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31, nwarps = nthr >> 5;
    if (TDT) {  // each warp its own copy: visible to its lanes after a warp sync
        if (lane < ND) s_dur[warp][lane] = m.durations[lane];
        __syncwarp();
    }
    long long sel_t0 = clock64();
    const int cur = par, nxt = par ^ 1;
#ifdef TBEAM_SEL_PAD
    {  // measurement: TBEAM_SEL_PAD straight-line ALU ops on warp 0's path (i-cache test)
        unsigned x = static_cast<unsigned>(clock()), y = static_cast<unsigned>(clock()) | 1u, z = y >> 3;
        unsigned x1 = x + 1, x2 = x + 2, x3 = x + 3;
#pragma unroll
        for (int q = 0; q < TBEAM_SEL_PAD / 4; ++q) {
            asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z));
            asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x1) : "r"(y), "r"(z));
            asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x2) : "r"(y), "r"(z));
            asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x3) : "r"(y), "r"(z));
        }
        if ((x ^ x1 ^ x2 ^ x3) == 0x12345u) st.g[1] = 0;
    }
#endif
    const bool last_round = r == cfg.token_rounds;
    const size_t S = st.S;
    const bool do_prefix = cfg.algo == 2 && cfg.prefix && r == 0 && (ND == 0 || m.di0 >= 0);

    // 1. slot state (warp 0, lane = slot) and counters: loaded into registers
    //    here, committed to shared memory after 2. -- the loads share 2.'s round
    //    trip instead of costing one of their own
    double p_sc = 0.0;
    unsigned long long p_hs = 0ull, p_ctr = 0ull;
    int p_ln = 0, p_ls = 0, p_f = 0, p_tn = 0, p_lm = 0, p_don = 0, p_pid = 0;
    if (tid < K) {
        const int s = b * K + tid;
        p_sc = st.score[s];
        p_f = st.f[s];
        p_ln = st.len[s];
        p_hs = st.hash[s];
        p_ls = st.last[s];
        p_tn = st.tnode[s];
        p_lm = st.lm_state[s];
        p_don = cfg.quirk ? st.sdonated[s] : 0;
        p_pid = st.pid[s];
    }
    if (tid >= 32 && tid < 37) p_ctr = st.ctr[static_cast<size_t>(b) * 5 + (tid - 32)];
    if (tid == 0) {
        n_edges = 0;
        n_final = 0;
        n_early = 0;
    }

    // 2. per slot (one warp): stage the NT partial records with one coalesced
    //    16-B pass issued before the activity test resolves; reduce them to
    //    the row normaliser and the top-K fused tokens; then (no prefix pass
    //    this round) write the slot's candidate region --------------------------
    const int NT = st.NT;
    const int ps = part_stride(K);
    // candidate region of slot i: [0, K) tokens, K + d the frame-leaving blank
    // column with duration index d (RNN-T: d = 0); lanes of the owning warp
    auto fill_cands = [&](int i, double base, int len_i, int f_i, int don_i, int tkn_i) {
        const long long sb = static_cast<long long>(i) * R * ndx;
        const int rb = i * RS;
        if constexpr (!TDT) {
            // RNN-T: one lane per entry (a second pass for K = 32's blank,
            // entry 32), predicated -- the token lanes and the blank lane take
            // no divergent paths
            #pragma unroll 1
            for (int e = lane; e < RS; e += 32) {
                const bool fin = base != -INFINITY, comp = f_i != t, isb = e == K;
                const int ec = e < K ? e : K - 1;
                const double tv = tkv[i * K + ec];
                const int tk = tki[i * K + ec];
                const double fb = fbl[i];
                const bool tokok = fin & !comp & !isb & (e < tkn_i) & !don_i & (len_i < cfg.max_len) & !last_round;
                const bool bl = fin & isb;
                csc[rb + e] = bl ? (comp ? base : base + fb) : (tokok ? tv + base : -INFINITY);
                cidx[rb + e] = bl ? sb + V : (tokok ? sb + tk : 0);
                ck[rb + e] = bl ? V : (tokok ? tk : -1);
                cdi[rb + e] = 0;
                cdest[rb + e] = bl ? (comp ? f_i : min(t + 1, T)) : (tokok ? t : 0);
            }
        } else {  // (compiled for TDT only)
        #pragma unroll 1
        for (int e = lane; e < RS; e += 32) {
            double v = -INFINITY;
            long long id = 0;
            int k = -1, d = 0, dest = 0;
            if (base != -INFINITY) {
                if (f_i != t) {  // complete: carry the slot with its blank column
                    if (e == K) {
                        v = base;
                        id = sb + static_cast<long long>(V) * ndx;
                        k = V;
                        dest = f_i;
                    }
                } else if (e >= K) {  // blank with duration index e - K
                    d = e - K;
                    if (ND == 0) {
                        if (d == 0) {
                            v = base + fbl[i];
                            id = sb + V;
                            k = V;
                            dest = min(t + 1, T);
                        }
                    } else if (d < ND && TDUR(d) >= 1) {  // blank must advance
                        v = base + (fbl[i] + dlp[i * ndx + d]);
                        id = sb + static_cast<long long>(V) * ndx + d;
                        k = V;
                        dest = min(t + TDUR(d), T);
                    }
                } else if (ND == 0 && e < tkn_i && !don_i && len_i < cfg.max_len && !last_round) {
                    v = tkv[i * K + e] + base;
                    id = sb + tki[i * K + e];
                    k = tki[i * K + e];
                    dest = t;
                }
            }
            if (ND > 0 && e < K) continue;  // TDT token entries below
            csc[rb + e] = v;
            cidx[rb + e] = id;
            ck[rb + e] = k;
            cdi[rb + e] = d;
            cdest[rb + e] = dest;
        }
        if (ND > 0) {
            // TDT: the slot's top-K (token, duration) combos (log p = lp_tok +
            // lp_dur; the last round of a frame admits d >= 1 only)
            int nsel = 0;
            if (base != -INFINITY && f_i == t && !don_i && len_i < cfg.max_len && tkn_i > 0) {
                double* cv = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(stg) + static_cast<size_t>(warp) * L.stg_per);
                long long* ckey = reinterpret_cast<long long*>(cv + tkn_i * ND);
                const int nc = tkn_i * ND;
                __syncwarp();
                #pragma unroll 1
                for (int e = lane; e < nc; e += 32) {
                    const int j = e / ND, d = e - j * ND;
                    const bool ok = !(last_round & (TDUR(d) == 0));
                    cv[e] = ok ? tkv[i * K + j] + dlp[i * ndx + d] : -INFINITY;
                    ckey[e] = sb + static_cast<long long>(tki[i * K + j]) * ndx + d;
                }
                __syncwarp();
                nsel = warp_select<NPRE>(cv, ckey, nc, K, pick + i * K);
            }
            #pragma unroll 1
            for (int q = lane; q < K; q += 32) {  // (predicated)
                const bool ok = q < nsel;
                const int e = ok ? pick[i * K + q] : 0;
                const int j = e / ND, d = e - j * ND;
                csc[rb + q] = ok ? base + (tkv[i * K + j] + dlp[i * ndx + d]) : -INFINITY;
                cidx[rb + q] = sb + static_cast<long long>(tki[i * K + j]) * ndx + d;
                ck[rb + q] = ok ? tki[i * K + j] : -1;
                cdi[rb + q] = d;
                cdest[rb + q] = min(t + TDUR(d), T);
            }
        }
        }
    };
    #pragma unroll 1
    for (int i = warp; i < K; i += L.cw) {
        if (warp >= L.cw) break;
        long long sub_t0 = clock64();
        const size_t s = static_cast<size_t>(b) * K + i;
        const double scv = st.score[s];
        const int fv = st.f[s];
        const int len_i = st.len[s];
        const int don_i = cfg.quirk ? st.sdonated[s] : 0;
        float* w = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(stg) + static_cast<size_t>(warp) * L.stg_per);
        int* heads = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(w) +
                                            stg_data_bytes(K, ndx, static_cast<size_t>(NT) * ps));
        const float4* src = reinterpret_cast<const float4*>(st.part + s * NT * ps);
        const int n4 = NT * ps / 4;
        const float blg = st.blank_logit[s];
        const float dv = (ND > 0 && lane < ND) ? st.dur_logit[s * ndx + lane] : -INFINITY;
        {
            int e = lane;
            for (; e + 96 < n4; e += 128) {
                const float4 a0 = src[e], a1 = src[e + 32], a2 = src[e + 64], a3 = src[e + 96];
                reinterpret_cast<float4*>(w)[e] = a0;
                reinterpret_cast<float4*>(w)[e + 32] = a1;
                reinterpret_cast<float4*>(w)[e + 64] = a2;
                reinterpret_cast<float4*>(w)[e + 96] = a3;
            }
            #pragma unroll 1
            for (; e < n4; e += 32) reinterpret_cast<float4*>(w)[e] = src[e];
        }
        int found = 0;
        // (a finished stream's rows were not scored this round: its staged
        // records are stale, so nothing below may index through them)
        if (!dn && scv != -INFINITY && fv == t) {
            __syncwarp();
            SUB_MARK(8);
            float mx = -INFINITY;
            #pragma unroll 1
            for (int q = lane; q < NT; q += 32) mx = fmaxf(mx, w[q * ps]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            // tile sums rescaled in fp32 (one ex2 each), reduced in fp64
            double sum = 0.0;
            #pragma unroll 1
            for (int q = lane; q < NT; q += 32) {
                const float pm = w[q * ps];
#if TBEAM_EXACT_EXP
                if (pm != -INFINITY) sum += static_cast<double>(w[q * ps + 1]) * exp(static_cast<double>(pm) - mx);
#else
                if (pm != -INFINITY) sum += static_cast<double>(w[q * ps + 1] * __expf(pm - mx));
#endif
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            const double lz = static_cast<double>(mx) + d_log(sum);
            const double ab = static_cast<double>(blg) - lz;
            const double l1 = ((LM && cfg.late) && cfg.blank_mode == 1) ? d_log1mexp(ab) : 0.0;
            SUB_MARK(9);
            if (ND > 0) {  // durations (TDT): own log-softmax
                float dm = dv;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) dm = fmaxf(dm, __shfl_xor_sync(0xffffffffu, dm, o));
                double de = lane < ND ? d_exp(static_cast<double>(dv) - dm) : 0.0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) de += __shfl_xor_sync(0xffffffffu, de, o);
                if (lane < ND) dlp[i * ndx + lane] = static_cast<double>(dv) - (static_cast<double>(dm) + d_log(de));
            }
            SUB_MARK(10);
            // top-K tokens: K-way merge of the NT per-tile lists
            if constexpr (KT == 1) {
                found = warp_merge_reg<1>(w, NT, ps, K, tki + i * K, tkv + i * K, edon + i * K);
            } else if constexpr (KT == 4) {
                found = warp_merge_reg<4>(w, NT, ps, K, tki + i * K, tkv + i * K, edon + i * K);
            } else if constexpr (KT == 8) {
                found = warp_merge_reg<8>(w, NT, ps, K, tki + i * K, tkv + i * K, edon + i * K);
            } else if constexpr (KT > 8) {
                found = warp_merge_lists(w, NT, ps, K, heads, tki + i * K, tkv + i * K, edon + i * K);
            } else {
                if (K == 1) found = warp_merge_reg<1>(w, NT, ps, K, tki + i * K, tkv + i * K, edon + i * K);
                else if (K <= 4) found = warp_merge_reg<4>(w, NT, ps, K, tki + i * K, tkv + i * K, edon + i * K);
                else if (K <= 8) found = warp_merge_reg<8>(w, NT, ps, K, tki + i * K, tkv + i * K, edon + i * K);
                else found = warp_merge_lists(w, NT, ps, K, heads, tki + i * K, tkv + i * K, edon + i * K);
            }
            SUB_MARK(11);
            // fused values of the winners (late fusion: the epilogue's LM-row
            // value, NGramLm::score_vocab's entry)
            if (lane < found) {
                const double lmv = (LM && cfg.late) ? edon[i * K + lane] : 0.0;
                tkv[i * K + lane] = fused_token(cfg, tkv[i * K + lane], lz, lmv, l1);
            }
            if (lane == 0) {
                lse[i] = lz;
                asrb[i] = ab;
                fbl[i] = fused_blank(cfg, ab);
                l1m[i] = l1;
            }
            __syncwarp();
        }
        if (lane == 0) tkn[i] = found;
        if (!do_prefix && !dn) fill_cands(i, scv, len_i, fv, don_i, found);
        __syncwarp();
        SUB_MARK(12);
    }
    SEL_MARK(13);
    // a finished stream stops here (uniform over the CTA): its loads above went
    // out with everyone's instead of behind the done flag, its writes were smem
    if (TB_UNLIKELY(dn)) return;
    if (tid < K) {
        sc[tid] = p_sc;
        ln[tid] = p_ln;
        hs[tid] = p_hs;
        ls[tid] = p_ls;
        fr[tid] = p_f;
        tn[tid] = p_tn;
        lmst[tid] = p_lm;
        act[tid] = (p_sc != -INFINITY && p_f == t) ? 1 : 0;
        don[tid] = p_don;
        s_pid[tid] = p_pid;
    }
    if (tid >= 32 && tid < 37) s_ctr[tid - 32] = p_ctr;
    __syncthreads();  // ---------------------------------------------- barrier 1
    SEL_MARK(1);

    // 3. AES++ maximum-length prefix combination (round 0 of a frame), then
    //    the candidate regions with the donations applied ---------------------
    if (TB_UNLIKELY(do_prefix)) {
        #pragma unroll 1
        for (int p = tid; p < K * K; p += nthr) {
            const int a = p / K, c = p % K;
            if (a == c || !act[a] || !act[c] || ln[c] != ln[a] + 1) continue;
            if (d_update_hash(hs[a], ls[c], cfg.hbase, cfg.hmod) == hs[c]) {
                const int e = atomicAdd(&n_edges, 1);
                ea[e] = a;
                ec[e] = c;
            }
        }
        __syncthreads();
        SEL_MARK(19);
        const int ne = n_edges;
        // sort by (len(receiver), receiver, donor): counting ranks over the
        // unique keys len<<10 | receiver<<5 | donor, one edge per thread (a
        // serial insertion sort of ~100 edges cost ~20k cycles at K = 16)
        // (scratch: edon, free until the donations below -- 2 K^2 ints)
        int* ekey = reinterpret_cast<int*>(edon);
        int* ekey2 = ekey + K * K;
        #pragma unroll 1
        for (int e = tid; e < ne; e += nthr) ekey[e] = (ln[ec[e]] << 10) | (ec[e] << 5) | ea[e];
        __syncthreads();
        #pragma unroll 1
        for (int e = tid; e < ne; e += nthr) {
            const int key = ekey[e];
            int rank = 0;
            #pragma unroll 4
            for (int f = 0; f < ne; ++f) rank += ekey[f] < key ? 1 : 0;
            ekey2[rank] = key & 0x3ff;  // receiver << 5 | donor
        }
        __syncthreads();
        #pragma unroll 1
        for (int e = tid; e < ne; e += nthr) {
            ea[e] = ekey2[e] & 31;
            ec[e] = ekey2[e] >> 5;
        }
        __syncthreads();
        SEL_MARK(20);
        // donor's fused value of the receiver's last token: z_a . W_out[last] + b
        #pragma unroll 1
        for (int e = warp; e < ne; e += nwarps) {
            const int a = ea[e], c = ec[e];
            const int k = ls[c];
            if (st.probe_on) {  // the joint epilogue's logit of column last[c] in slot a's row
                if (lane == 0) {
                    const double logit = static_cast<double>(st.probe[(static_cast<size_t>(b) * K + a) * K + c]);
                    const double lmv = (LM && cfg.late) ? lm_vocab_value(lm, lmst[a], k) : 0.0;
                    double part = fused_token(cfg, logit, lse[a], lmv, l1m[a]);
                    if (ND > 0) part += dlp[a * ndx + m.di0];
                    if ((LM && cfg.early)) {
                        double term = lm_score_token(lm, lmst[a], k);
                        if (cfg.blank_mode == 1) term += d_log1mexp(asrb[a]);
                        part += cfg.lam * term;
                    }
                    edon[e] = part;
                }
                continue;
            }
            // (no shortcut through this round's z16 rows: other streams' select
            // CTAs are already staging the next round's operands over them)
            const float* ep = st.encp + (static_cast<size_t>(b) * st.Tmax + t) * m.J;
            const float* pp = st.pred + (static_cast<size_t>(b) * st.P + s_pid[a]) * m.J;
            // (unrolled: TBEAM_DONOR_UNROLL iterations' loads go out together --
            // the encoder row is DRAM-cold, so each batch is a full round trip;
            // the per-lane accumulation order is unchanged)
            float acc = 0.f;
            const bool bfp = m.prec == 1;
            #pragma unroll kDonorUnroll
            for (int j = lane; j < m.J; j += 32) {
                const float e = __ldg(ep + j), p = __ldg(pp + j);
                const float wv = bfp ? __bfloat162float(m.w_out16[static_cast<size_t>(k) * m.J + j])
                                     : __ldg(m.w_out + static_cast<size_t>(k) * m.J + j);
                float z = tanhf(e + p);
                if (bfp) z = bf16_round(z);
                acc = fmaf(z, wv, acc);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) {
                const double logit = static_cast<double>(acc + m.b_out[k]);
                const double lmv = (LM && cfg.late) ? lm_vocab_value(lm, lmst[a], k) : 0.0;
                double part = fused_token(cfg, logit, lse[a], lmv, l1m[a]);
                if (ND > 0) part += dlp[a * ndx + m.di0];
                if ((LM && cfg.early)) {
                    double term = lm_score_token(lm, lmst[a], k);
                    if (cfg.blank_mode == 1) term += d_log1mexp(asrb[a]);
                    part += cfg.lam * term;
                }
                edon[e] = part;
            }
        }
        __syncthreads();
        SEL_MARK(21);
        if (tid == 0) {  // serial application in sorted order
            #pragma unroll 1
            for (int e = 0; e < ne; ++e) {
                const int a = ea[e], c = ec[e];
#ifdef TBEAM_DEBUG_PREFIX
                if (b == 0 && t == TBEAM_DEBUG_PREFIX)
                    printf("GPU prefix t=%d edge %d->%d last=%d sc_a=%.9f sc_c=%.9f don=%.9f lse=%.9f l1m=%.9f lm_st=%d\n", t, a, c,
                           ls[c], sc[a], sc[c], edon[e], lse[a], l1m[a], lmst[a]);
#endif
                sc[c] = d_merge(sc[c], sc[a] + edon[e], cfg.merge_mode);
                don[a] = 1;
            }
            if ((LM && cfg.early)) n_early += ne;
        }
        __syncthreads();
        SEL_MARK(22);
        if (TB_UNLIKELY((st.trace & 1) && tid == 0)) s_sel_tr[23] += ne;
        // (only the L.cw staging warps own a scratch area for the TDT combos)
        if (warp < L.cw) {
            #pragma unroll 1
            for (int i = warp; i < K; i += L.cw) fill_cands(i, sc[i], ln[i], fr[i], don[i], tkn[i]);
        }
        __syncthreads();
    }
    SEL_MARK(2);

    // 4. recombination of the frame-leaving blank column by (HypKey, dest):
    //    the first of each group (in slot-major order) log-adds the later ones;
    //    5. prune_topk: top-K by (score desc, index asc).  Both by warp 0 (the
    //    other warps go on to barrier 4): warp syncs instead of CTA barriers
    const int nb = K * ndx;
    const int total = K * RS;
    if (warp == 0) {
        if constexpr (!TDT) {
            // RNN-T: one blank entry per slot -- lane i compares its key
            // (hash, length, last, destination) with every slot's in one pass:
            // an earlier equal finite entry makes it a non-leader, later ones
            // are log-added in slot order
            if (lane < K) {
                const int e = lane * RS + K;
                const double cv = csc[e];
                const unsigned long long h = hs[lane];
                const int l = ln[lane], z = ls[lane], dest = cdest[e];
                unsigned later = 0u;
                bool leader = true;
                #pragma unroll 1
                for (int j = 0; j < K; ++j) {
                    const int ej = j * RS + K;
                    const bool same = (j != lane) & (csc[ej] != -INFINITY) & (hs[j] == h) & (ln[j] == l) &
                                      (ls[j] == z) & (cdest[ej] == dest);
                    leader &= !(same & (j < lane));
                    later |= (same & (j > lane)) ? 1u << j : 0u;
                }
                double accv = cv;
                if (cv != -INFINITY) {
                    if (!leader) {
                        accv = -INFINITY;
                    } else {
                        #pragma unroll 1
                        while (later) {
                            const int j = __ffs(later) - 1;
                            later &= later - 1u;
                            accv = d_merge(accv, csc[j * RS + K], cfg.merge_mode);
                        }
                    }
                }
                nsc[lane] = accv;
            }
        } else {
            // slot level first: lane i < K collects the other slots with the same
            // (hash, length, last token); entry x = (slot i, duration x % ndx) then
            // only compares against the entries of those slots and its own (equal
            // destinations: frames clipped at T).  Ascending scan = slot-major
            // order: an earlier equal entry makes x a non-leader, later ones are
            // log-added in order.
            unsigned dupm = 0u;
            if (lane < K) {
                const unsigned long long h = hs[lane];
                const int l = ln[lane], z = ls[lane];
                #pragma unroll 1
                for (int j = 0; j < K; ++j)
                    dupm |= ((hs[j] == h) & (ln[j] == l) & (ls[j] == z) & (j != lane)) ? 1u << j : 0u;
                s_dupm[lane] = dupm;
            }
            __syncwarp();
            #pragma unroll 1
            for (int x = lane; x < nb; x += 32) {
                const int i = x / ndx, e = i * RS + K + (x - i * ndx);
                const double cv = csc[e];
                double accv = cv;
                if (cv != -INFINITY) {
                    const int dest = cdest[e];
                    unsigned mm = s_dupm[i] | (1u << i);
                    bool leader = true;
                    #pragma unroll 1
                    while (mm && leader) {
                        const int j = __ffs(mm) - 1;
                        mm &= mm - 1u;
                        #pragma unroll 1
                        for (int dd = 0; dd < ndx; ++dd) {
                            const int y = j * ndx + dd;
                            const int ey = j * RS + K + dd;
                            const double cy = csc[ey];
                            const bool eq = (y != x) & (cy != -INFINITY) & (cdest[ey] == dest);
                            if (eq) {  // rare: equal keys (same slot: destinations clipped at T)
                                if (y < x) {
                                    leader = false;
                                    break;
                                }
                                accv = d_merge(accv, cy, cfg.merge_mode);
                            }
                        }
                    }
                    if (!leader) accv = -INFINITY;
                }
                nsc[x] = accv;
            }
        }
        __syncwarp();
#ifdef TBEAM_DEBUG_PREFIX
        if (b == 0 && t == TBEAM_DEBUG_PREFIX && lane == 0)
            for (int x = 0; x < nb; ++x) {
                const int i = x / ndx, e = i * RS + K + (x - i * ndx);
                if (csc[e] != -INFINITY)
                    printf("GPU blank t=%d r=%d slot %d d %d dest %d before %.9f after %.9f\n", t, r, i, x - i * ndx,
                           cdest[e], csc[e], nsc[x]);
            }
        if (b == 0 && t == TBEAM_DEBUG_PREFIX && lane == 0)
            for (int x = 0; x < total; ++x)
                if (csc[x] != -INFINITY && (x % RS) < K)
                    printf("GPU token t=%d r=%d slot %d k %d v %.9f\n", t, r, x / RS, ck[x], csc[x]);
#endif
        #pragma unroll 1
        for (int x = lane; x < nb; x += 32) csc[(x / ndx) * RS + K + (x % ndx)] = nsc[x];
        __syncwarp();
        SEL_MARK(14);
        const int f = total <= 32 ? warp_rank<1>(csc, cidx, total, K, sel)
                                  : warp_pruned_rank(csc, cidx, total, K, RS, sel, reinterpret_cast<unsigned char*>(stg));
        if (lane == 0) n_final = f;
        SEL_MARK(15);
    }
    SEL_MARK(3);

    // 6. expansion (warp 0, lane = new slot j): hyp_store.cpp:89-135,
    //    decoder.cpp:282-324; then the stream's state machine ---------------
    if (warp == 0) {
        __syncwarp();
        const int F = min(n_final, K);
        double n_score = -INFINITY;
        int n_len = 0, n_last = -1, n_f = T, n_tn = -1, n_lm = 0, n_par = 0, n_tok = -1;
        unsigned long long n_hash = 0ull;
        int early_j = 0;
        if (lane < K) {
            const int j = lane;
            const int sout = b * K + j;
            if (j < F) {
                const int x = sel[j];
                const int p = x / RS;
                const int k = ck[x];
                double s = csc[x];
                n_par = p;
                if (k == V) {
                    n_len = ln[p];
                    n_hash = hs[p];
                    n_last = ls[p];
                    n_tn = tn[p];
                    n_lm = lmst[p];
                    n_f = cdest[x];
                } else {
                    if ((LM && cfg.early)) {
                        double term = lm_score_token(lm, lmst[p], k);
                        if (cfg.blank_mode == 1) term += d_log1mexp(asrb[p]);
                        s += cfg.lam * term;
                        early_j = 1;
                    }
                    n_len = ln[p] + 1;
                    n_hash = d_update_hash(hs[p], k, cfg.hbase, cfg.hmod);
                    n_last = k;
                    n_f = cdest[x];
                    n_lm = (LM && cfg.with_lm) ? lm_advance(lm, lmst[p], k) : 0;
                    n_tok = k;
                    if (col < st.max_cols) {
                        const size_t node = static_cast<size_t>(col) * S + sout;
                        st.st_tok[node] = k;
                        st.st_prev[node] = tn[p];
                        st.st_dur[node] = ND > 0 ? static_cast<signed char>(TDUR(cdi[x])) : 0;
                        n_tn = static_cast<int>(node);
                    } else {
                        n_tn = -2;  // trie overflow (guarded on the host by max_cols)
                    }
                }
                n_score = sc[p] + (s - sc[p]);
            } else {
                n_par = 0;
                n_len = ln[0];
                n_hash = hs[0];
                n_last = ls[0];
                n_tn = tn[0];
                n_lm = lmst[0];
            }
            s_par[j] = n_par;
            s_tok[j] = n_tok;
        }
        SEL_MARK(16);
        if (lane == 0 && col < st.max_cols) st.st_frame[static_cast<size_t>(col) * st.B + b] = t;
        const int n_active = __popc(__ballot_sync(0xffffffffu, lane < K && act[lane]));
        const int n_early_r = __popc(__ballot_sync(0xffffffffu, early_j != 0));
        // prediction-state pool (2K entries per stream): a blank / dead child
        // keeps its parent's entry (no copy); the q-th token child takes the
        // q-th lowest entry no current slot uses, so the parent's state stays
        // intact for this round's LSTM step
        const unsigned long long pbit = lane < K ? (1ull << s_pid[lane]) : 0ull;
        const unsigned long long used =
            static_cast<unsigned long long>(__reduce_or_sync(0xffffffffu, static_cast<unsigned>(pbit >> 32))) << 32 |
            __reduce_or_sync(0xffffffffu, static_cast<unsigned>(pbit));
        const bool tokchild = lane < K && n_tok >= 0;
        const unsigned tkb = __ballot_sync(0xffffffffu, tokchild);
        int npid = 0;
        if (tokchild) {
            unsigned long long fr = ~used;
            #pragma unroll 1
            for (int q = __popc(tkb & ((1u << lane) - 1u)); q > 0; --q) fr &= fr - 1ull;
            npid = __ffsll(static_cast<long long>(fr)) - 1;
        } else if (lane < K) {
            npid = s_pid[n_par];
        }
        SEL_MARK(17);
        // stream state machine (decoder.cpp:143-158) + counters
        const bool alive_here = lane < K && n_score != -INFINITY && n_f == t;
        const bool any = __ballot_sync(0xffffffffu, alive_here) != 0u;
        const int fmin = __reduce_min_sync(0xffffffffu, (lane < K && n_score != -INFINITY) ? n_f : T);
        int nr = r + 1, nt = t, newframe = 0;
        if (nr >= cfg.rounds || !any) {
            nt = fmin;
            if (nt <= t) nt = t + 1;
            nr = 0;
            newframe = 1;
        }
        const int done = nt >= T ? 1 : 0;
        SEL_MARK(18);
        // token rows of the LSTM step and next round's joint rows: one
        // warp-aggregated atomic per list, both in flight together
        const unsigned tbal = LSTM ? tkb : 0u;
        const bool nact = lane < K && !done && n_score != -INFINITY && n_f == nt;
        const unsigned abal = __ballot_sync(0xffffffffu, nact);
        int ubase = 0, abase = 0;
        if (lane == 0) {
            if (tbal) ubase = atomicAdd(&st.upd_count[cur], __popc(tbal));
            if (abal) abase = atomicAdd(&st.act_count[nxt], __popc(abal));
        }
        SEL_MARK(4);
        if (lane == 0) {
            unsigned long long* gctr = st.ctr + static_cast<size_t>(b) * 5;
            const int ne = n_early + n_early_r;
            gctr[0] = s_ctr[0] + (newframe ? 1ull : 0ull);
            gctr[1] = s_ctr[1] + 1ull;
            gctr[2] = s_ctr[2] + static_cast<unsigned long long>(n_active);
            gctr[3] = s_ctr[3] + static_cast<unsigned long long>(ne);
            gctr[4] = s_ctr[4] + ((LM && cfg.late) ? static_cast<unsigned long long>(n_active) : 0ull);
            if (done) {
                st.steps[b] = col + 1;
                atomicAdd(st.n_done, 1);
            }
            st.col[b] = col + 1;
            st.t[b] = nt;
            st.r[b] = nr;
            st.done[b] = done;
            s_t = nt;
            s_done = done;
        }
        // the new beam's slot state + the compacted rows
        ubase = __shfl_sync(0xffffffffu, ubase, 0);
        abase = __shfl_sync(0xffffffffu, abase, 0);
        if (lane < K) {
            const int j = lane;
            const size_t s = static_cast<size_t>(b) * K + j;
            int upos = -1;
            if ((tbal >> j) & 1u) {
                upos = ubase + __popc(tbal & ((1u << j) - 1u));
                st.upd_list[cur * S + upos] = static_cast<int>(s);
                st.upd_src[cur * S + upos] = b * st.P + s_pid[n_par];
                st.upd_dst[cur * S + upos] = b * st.P + npid;
                st.upd_tok[cur * S + upos] = n_tok;
            }
            if (st.tc) st.upd_pos[s] = upos;
            s_upos[j] = upos;
            s_npid[j] = npid;
            st.score[s] = n_score;
            st.len[s] = n_len;
            st.hash[s] = n_hash;
            st.last[s] = n_last;
            st.f[s] = n_f;
            st.tnode[s] = n_tn;
            st.lm_state[s] = n_lm;
            st.pid[s] = npid;
            // aes_pp quirk: per-slot flag, not permuted, reset at frame start only
            st.sdonated[s] = (cfg.quirk && !newframe) ? static_cast<unsigned char>(don[j]) : 0;
            int apos = -1;
            if (nact) {
                apos = abase + __popc(abal & ((1u << j) - 1u));
                st.act_list[nxt * S + apos] = static_cast<int>(s);
            }
            if (st.tc) st.act_pos[s] = apos;
            s_apos[j] = apos;
        }
    }
    __syncthreads();  // ---------------------------------------------- barrier 4
    if (TB_UNLIKELY(s_done)) return;

    SEL_MARK(5);
    // 9. prediction-network state of the new beam, gathered by parent (decoder.cpp
    //    :288-318): blank/dead children copy the parent's state; token children
    //    shift the stateless window (model.cpp:109-121) or -- LSTM -- stage the
    //    parent's h for the gate GEMM.  Every slot active next round also gets
    //    its joint operand z = bf16(tanh(enc_proj[b, t'] + pred)) (tensor-core path).
    const float* ep = st.encp + (static_cast<size_t>(b) * st.Tmax + s_t) * m.J;
    const size_t prow0 = static_cast<size_t>(b) * st.P;  // this stream's pool rows
    if (LSTM) {
        // token children: stage the parent's h (bf16) for the gate GEMM;
        // children active next round that keep their entry: z = tanh(enc + pred).
        // Items go in batches of TBEAM_STAGE_BATCH (4) per thread: every global load of a batch is
        // issued before the first use (read-only data: __ldg), one round trip
        // per batch instead of one per item.
        const int H4 = m.H >> 2, J4 = m.J >> 2;
        const int W4 = H4 > J4 ? H4 : J4;
        const int nitems = K * W4;
        #pragma unroll 1
        for (int base = tid; base < nitems; base += TBEAM_STAGE_BATCH * nthr) {
            float4 va[TBEAM_STAGE_BATCH], vb[TBEAM_STAGE_BATCH];
            int kind[TBEAM_STAGE_BATCH], dsto[TBEAM_STAGE_BATCH];
#pragma unroll
            for (int u = 0; u < TBEAM_STAGE_BATCH; ++u) {
                const int it = base + u * nthr;
                kind[u] = 0;
                dsto[u] = 0;
                if (it < nitems) {
                    const int j = it / W4, e = it - j * W4;
                    if (s_tok[j] >= 0) {
                        if (st.tc && e < H4) {
                            kind[u] = 1;
                            va[u] = __ldg(reinterpret_cast<const float4*>(st.h + (prow0 + s_pid[s_par[j]]) * m.H) + e);
                            dsto[u] = s_upos[j] * st.Hp + 4 * e;
                        }
                    } else if (st.tc && s_apos[j] >= 0 && e < J4) {
                        kind[u] = 2;
                        va[u] = __ldg(reinterpret_cast<const float4*>(st.pred + (prow0 + s_npid[j]) * m.J) + e);
                        vb[u] = __ldg(reinterpret_cast<const float4*>(ep) + e);
                        dsto[u] = s_apos[j] * st.Jp + 4 * e;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < TBEAM_STAGE_BATCH; ++u) {
                if (kind[u] == 0) continue;
                const float4 v = va[u];
                if (kind[u] == 1) {
                    put_op4(st.hA16 + dsto[u], st.hpl, st.split3, v.x, v.y, v.z, v.w);
                } else {
                    const float4 ev = vb[u];
                    put_op4(st.z16 + dsto[u], st.zpl, st.split3, tanhf(ev.x + v.x), tanhf(ev.y + v.y),
                            tanhf(ev.z + v.z), tanhf(ev.w + v.w));
                }
            }
        }
        return;
    }
    // stateless: a token child's window = parent's window shifted + token
    // (model.cpp:109-121) and pred = b + (1/n) sum table[w], in its new entry
    const int n = m.n;
    __shared__ int s_win[kMaxBeam * 16];
    const bool win_smem = n <= 16;
    if (tid < K && s_tok[tid] >= 0) {
        const int j = tid, tok = s_tok[j];
        const int* wsrc = st.win + (prow0 + s_pid[s_par[j]]) * n;
        int* wdst = st.win + (prow0 + s_npid[j]) * n;
        #pragma unroll 1
        for (int q = 0; q < n; ++q) {
            const int w = q + 1 < n ? wsrc[q + 1] : tok;
            wdst[q] = w;
            if (win_smem) s_win[j * 16 + q] = w;
        }
    }
    __syncthreads();
    const float inv = n > 0 ? 1.0f / n : 0.f;
    #pragma unroll 1
    for (int it = tid; it < K * m.J; it += nthr) {
        const int j = it / m.J, c = it - j * m.J;
        const int tok = s_tok[j], apos = s_apos[j];
        if (tok < 0 && !(st.tc && apos >= 0)) continue;
        const size_t row = prow0 + s_npid[j];
        float v;
        if (tok < 0) {
            v = st.pred[row * m.J + c];
        } else {
            float acc = 0.f;
            const int* wl = st.win + row * n;
            #pragma unroll 1
            for (int q = 0; q < n; ++q) {
                const int w = win_smem ? s_win[j * 16 + q] : wl[q];
                acc += inv * m.table[static_cast<size_t>(w < 0 ? m.V : w) * m.J + c];
            }
            v = m.b_pred[c] + acc;
            st.pred[row * m.J + c] = v;
        }
        if (st.tc && apos >= 0) put_op(st.z16 + static_cast<size_t>(apos) * st.Jp + c, st.zpl, st.split3, tanhf(ep[c] + v));
    }
}

// One CTA (256 threads) per stream; the last CTA to finish does the loop
// bookkeeping: list-count resets for the parity double buffers, the round
// counter, and (set_cond) the CUDA-graph WHILE condition "a stream is still
// decoding" -- so the loop needs no control kernel and no host sync.
template <bool LSTM, bool TDT, bool LM, int KT>
__global__ void __launch_bounds__(256) select_kernel(DevModel m, DevLm lm, DevCfg cfg, DevState st, SelSmem L,
                                                     int par, cudaGraphConditionalHandle hcond, int set_cond) {
    const bool tlon = (st.trace & 2) && threadIdx.x == 0;
    const unsigned long long tl_entry = tlon ? gtimer() : 0ull;
    pdl_trigger();
    pdl_wait();
    const unsigned long long tl_rel = tlon ? gtimer() : 0ull;
    const int tl_round = tlon ? *st.g : -1;
    const long long tk0 = clock64();
    if (TB_UNLIKELY((st.trace & 1) && threadIdx.x < kSelTr)) s_sel_tr[threadIdx.x] = 0;
    __syncthreads();
    {
        // the stream's scalars in one batch of loads (col = its trie column =
        // its round count; t = frame, r = round in the frame)
        const int b = blockIdx.x;
        const int dn = st.done[b], col = st.col[b], t = st.t[b], r = st.r[b], T = st.T[b];
        select_stream<LSTM, TDT, LM, KT>(m, lm, cfg, st, L, par, col, t, r, T, dn);
    }
    const long long tk1 = clock64();
    if (TB_UNLIKELY(tlon)) tl_record(g_tl_sel, tl_round, 3, tl_entry, tl_rel, gtimer());
    if (threadIdx.x == 0) {
        if (blockIdx.x == 0) {
            st.act_count[par] = 0;      // read by this round's joint (finished)
            st.upd_count[par ^ 1] = 0;  // read by last round's LSTM GEMMs (finished)
        }
        // the round's bookkeeping: here (last CTA) unless the LSTM projection
        // GEMM -- the round's final kernel -- does it without fence / atomics
        const int k = st.round_in_proj ? 0 : (__threadfence(), atomicAdd(st.sel_blocks, 1));
        if (!st.round_in_proj && k == static_cast<int>(gridDim.x) - 1) {
            *st.sel_blocks = 0;
            const int inc = *st.live ? 1 : 0;
            const int rounds = atomicAdd(st.g, inc) + inc;
            const int nd = atomicAdd(st.n_done, 0);
            if (set_cond) cudaGraphSetConditional(hcond, (nd < st.B && rounds < st.max_cols) ? 1u : 0u);
        }
        if (TB_UNLIKELY((st.trace & 1) && blockIdx.x < kSelTraceCtas && !st.done[blockIdx.x])) {
            long long* g = g_sel_trace + blockIdx.x * kSelTr;
            g[0] += 1;
            for (int k = 1; k < 6; ++k) g[k] += s_sel_tr[k];
            for (int k = 8; k < kSelTr; ++k) g[k] += s_sel_tr[k];
            g[6] += clock64() - tk1;
            g[7] += tk1 - tk0;
        }
    }
}

// ---------------------------------------------------------------------------
// finalize: EOS (decoder.cpp:329-338), rank (score desc, slot asc), n-best
// backtrace through the token trie with alignments.  grid B, block 32.
// ---------------------------------------------------------------------------
__global__ void finalize_kernel(DevModel m, DevLm lm, DevCfg cfg, DevState st) {
    const int b = blockIdx.x;
    const int K = cfg.K;
    __shared__ int order[kMaxBeam];
    __shared__ int nalive;
    if (threadIdx.x == 0) {
        // final recombination (merge_duplicates_stream, hyp_store.cpp:169-191):
        // no-op for RNN-T; TDT tokens that jump to T_b arrive unmerged
        for (int i = 0; i < K; ++i) {
            const size_t si = static_cast<size_t>(b) * K + i;
            if (st.score[si] == -INFINITY) continue;
            for (int j = i + 1; j < K; ++j) {
                const size_t sj = static_cast<size_t>(b) * K + j;
                if (st.score[sj] == -INFINITY) continue;
                if (st.hash[si] == st.hash[sj] && st.len[si] == st.len[sj] && st.last[si] == st.last[sj]) {
                    st.score[si] = d_merge(st.score[si], st.score[sj], cfg.merge_mode);
                    st.score[sj] = -INFINITY;
                }
            }
        }
        int na = 0;
        for (int i = 0; i < K; ++i) {
            const size_t s = static_cast<size_t>(b) * K + i;
            double v = st.score[s];
            if (v == -INFINITY) continue;
            if (cfg.with_lm && cfg.eos) {
                v += cfg.lam * lm_score_eos(lm, st.lm_state[s]);
                st.score[s] = v;
                st.ctr[static_cast<size_t>(b) * 5 + 3] += 1ull;
            }
            order[na++] = i;
        }
        for (int x = 1; x < na; ++x) {  // insertion sort: score desc, slot asc
            const int a = order[x];
            const double va = st.score[static_cast<size_t>(b) * K + a];
            int y = x - 1;
            while (y >= 0) {
                const double vy = st.score[static_cast<size_t>(b) * K + order[y]];
                if (vy > va || (vy == va && order[y] < a)) break;
                order[y + 1] = order[y];
                --y;
            }
            order[y + 1] = a;
        }
        nalive = na;
        st.out_count[b] = min(na, cfg.nbest);
    }
    __syncthreads();
    const int take = min(nalive, cfg.nbest);
    for (int q = threadIdx.x; q < cfg.nbest; q += blockDim.x) {
        const size_t e = static_cast<size_t>(b) * cfg.nbest + q;
        if (q >= take) {
            st.out_len[e] = 0;
            st.out_score[e] = -INFINITY;
            continue;
        }
        const size_t s = static_cast<size_t>(b) * K + order[q];
        const int L = st.len[s];
        st.out_len[e] = L;
        st.out_score[e] = st.score[s];
        int node = st.tnode[s];
        for (int u = L - 1; u >= 0 && node >= 0; --u) {
            const size_t o = e * cfg.max_len + u;
            st.out_tok[o] = st.st_tok[node];
            st.out_frame[o] = st.st_frame[static_cast<size_t>(node / st.S) * st.B + b];
            st.out_dur[o] = st.st_dur[node];
            node = st.st_prev[node];
        }
    }
}

// ---- launchers ---------------------------------------------------------------

void tl_read_sel(int enable, unsigned long long* out) {
    if (out) cudaMemcpyFromSymbol(out, g_tl_sel, sizeof(unsigned long long) * kTlRounds * 16);
    unsigned long long* init = new unsigned long long[static_cast<size_t>(kTlRounds) * 16];
    for (size_t i = 0; i < static_cast<size_t>(kTlRounds) * 16; ++i) init[i] = (i % 4 == 0 || i % 4 == 1) ? ~0ull : 0ull;
    cudaMemcpyToSymbol(g_tl_sel, init, sizeof(unsigned long long) * kTlRounds * 16);
    delete[] init;
}

void sel_trace(int enable, long long* out) {
    if (out) cudaMemcpyFromSymbol(out, g_sel_trace, sizeof(long long) * kSelTraceCtas * kSelTr);
    static long long z[kSelTraceCtas * kSelTr] = {};
    cudaMemcpyToSymbol(g_sel_trace, z, sizeof(z));
}

// every (LSTM, TDT, LM) x beam specialisation: KT = 1, 8, 16 or 0 (any K)
// (K = 4 runs the any-K kernel: measured 0.6 us/round faster than its
// specialisation at the bench shape, which K = 1 and 8 gain 2.5 / 0.4 us from)
#define TBEAM_SEL_FOR_K(X, A, B, C) X(A, B, C, 0); X(A, B, C, 1); X(A, B, C, 8); X(A, B, C, 16)
#define TBEAM_SEL_FOR_ALL(X)                                                                      \
    TBEAM_SEL_FOR_K(X, true, true, true); TBEAM_SEL_FOR_K(X, true, true, false);                  \
    TBEAM_SEL_FOR_K(X, true, false, true); TBEAM_SEL_FOR_K(X, true, false, false);                \
    TBEAM_SEL_FOR_K(X, false, true, true); TBEAM_SEL_FOR_K(X, false, true, false);                \
    TBEAM_SEL_FOR_K(X, false, false, true); TBEAM_SEL_FOR_K(X, false, false, false)

void configure_kernels() {
#define TBEAM_SEL_ATTR(A, B, C, KT) \
    cudaFuncSetAttribute(select_kernel<A, B, C, KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)
    TBEAM_SEL_FOR_ALL(TBEAM_SEL_ATTR);
#undef TBEAM_SEL_ATTR
}

void launch_init(const DevModel& m, const DevLm& lm, const DevCfg& cfg, const DevState& st,
                 cudaStream_t s) {
    init_kernel<<<st.B, 128, 0, s>>>(m, lm, cfg, st);
}

void launch_select(const DevModel& m, const DevLm& lm, const DevCfg& cfg, const DevState& st, int par,
                   cudaGraphConditionalHandle h, int set_cond, cudaStream_t s) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(st.B);
    lc.blockDim = dim3(select_threads(cfg.K));
    const SelSmem L(cfg.K, m.ND > 0 ? st.ndx : 1, st.NT * part_stride(cfg.K), select_threads(cfg.K) / 32);
    lc.dynamicSmemBytes = L.total;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    const bool lstm = m.pred_kind == 1, tdt = m.ND > 0, lmx = cfg.with_lm != 0;
    int kt = cfg.K == 1 || cfg.K == 8 || cfg.K == 16 ? cfg.K : 0;
    if (const char* e = std::getenv("TBEAM_SEL_GENERIC"))  // measurement override: beams listed run the any-K kernel
        for (const char* q = e; *q; ++q)
            if (std::atoi(q) == cfg.K && (q == e || q[-1] == ',')) kt = 0;
#define TBEAM_SEL_KT(A, B, C, KT) \
    if (kt == KT) cudaLaunchKernelEx(&lc, select_kernel<A, B, C, KT>, m, lm, cfg, st, L, par, h, set_cond)
#define TBEAM_SEL(A, B, C)                         \
    do {                                           \
        TBEAM_SEL_FOR_K(TBEAM_SEL_KT, A, B, C);    \
    } while (0)
    if (lstm) {
        if (tdt) { if (lmx) TBEAM_SEL(true, true, true); else TBEAM_SEL(true, true, false); }
        else { if (lmx) TBEAM_SEL(true, false, true); else TBEAM_SEL(true, false, false); }
    } else {
        if (tdt) { if (lmx) TBEAM_SEL(false, true, true); else TBEAM_SEL(false, true, false); }
        else { if (lmx) TBEAM_SEL(false, false, true); else TBEAM_SEL(false, false, false); }
    }
#undef TBEAM_SEL
#undef TBEAM_SEL_KT
}

void launch_enc_to_bf16(const DevModel& m, const DevState& st, int rows, cudaStream_t s) {
    enc_to_bf16_kernel<<<148 * 8, 256, 0, s>>>(m, st, rows);
}

void launch_finalize(const DevModel& m, const DevLm& lm, const DevCfg& cfg, const DevState& st,
                     cudaStream_t s) {
    finalize_kernel<<<st.B, 32, 0, s>>>(m, lm, cfg, st);
}

}  // namespace tbeam_dev
