// CUDA-core (FFMA) GEMM kernels of the decode step, sm_100a.
//
//   enc_proj_simt    encoder projection  [B*T, D] x W_enc^T        (once per decode)
//   joint_simt       joint network on the compacted active rows, fused with the
//                    bias, the per-tile log-softmax statistics, late-pruning LM
//                    fusion and the per-row top-K     (ToyModel::score_row,
//                    model.cpp:337-367; selection_row decoder.cpp:47-61)
//   lstm_gates_simt  LSTM step of the token-emitting rows, gathered by parent
//   lstm_proj_simt   prediction projection of the same rows
//
// These are the CUDA-core fp32 path (precision = fp32 with TBEAM_FP32_SIMT=1;
// the default fp32 path is the tensor cores on three-plane operand splits,
// kernels_tc.cu tc_gemm_s3): fp32 operands and FFMA, partial sums of 8
// products folded into fp64 accumulators -- not TF32 -- so the scores stay
// within 1e-4 of the fp64 oracle; also the fallback of the bf16 path
// (operands rounded to bf16 exactly like the tensor-core kernels).  The
// encoder projection (once per decode) serves both fp32 paths.
// Thread layout of every tile: 256 threads, 32 rows x TCOLS columns, thread
// (ty, tx) owns rows 4ty..4ty+3 and columns tx, tx+32, ...  The decode-loop
// kernels use 32-column tiles (joint, projection) and 8-unit gate tiles:
// their GEMMs are latency-bound at decode row counts, so four times the CTAs
// of 128-column tiles finish ~4x sooner; the one-off encoder projection keeps
// 128-column tiles.
#include <cuda_bf16.h>

#include "device_fns.cuh"
#include "engine.cuh"
#include "kernels.h"

namespace tbeam_dev {

// Accumulation in the CUDA-core tiles.  The fp32 precision mode's contract is
// scores within 1e-4 of the fp64 oracle, and a plain fp32 accumulator over
// J = 640 products drifts past it on long streams.  Measured at C2 (T = 500,
// 16 streams, max |dscore| vs the oracle; us per round) -- DESIGN.md §3:
//   TBEAM_SIMT_ACC64=0  fp32 FFMA chain                      3.0e-4   111
//   TBEAM_SIMT_ACC64=1  fp64 DFMA                            1.3e-5   216
//   TBEAM_SIMT_ACC64=2  fp32 sums of TBEAM_FOLD products
//                       folded into fp64: FOLD 32            7.8e-5   117
//                                         FOLD 8 (default)   3.2e-5   120
// Accurate expf in the joint's tile sums (TBEAM_EXACT_EXP) is a measurement
// switch with no effect on the C2 error.
#ifndef TBEAM_SIMT_ACC64
#define TBEAM_SIMT_ACC64 2
#endif
#ifndef TBEAM_EXACT_EXP
#define TBEAM_EXACT_EXP 0
#endif
#ifndef TBEAM_FOLD
#define TBEAM_FOLD 8
#endif
#if TBEAM_SIMT_ACC64
using acc_t = double;
#else
using acc_t = float;
#endif

constexpr int TR = 32;   // rows per tile
constexpr int TC = 128;  // columns per tile
// k chunk (64 for the 32-column tiles measured 4% slower on C2)
template <int TCOLS>
__host__ __device__ constexpr int tk_for() { return TCOLS > 0 ? 32 : 32; }

// ---------------------------------------------------------------------------
// generic tile: acc[4][4] = A[rows] . W[cols]^T over Kd, A/W staged in smem
// ---------------------------------------------------------------------------
// Register double buffer: the next k-chunk's operands are fetched into
// registers (raw loads only) before the current chunk's FMAs, so every global
// round trip overlaps compute; afin turns a fetched A pair into the operand
// (e.g. tanh(enc + pred)) when it is written to shared memory.
template <int TCOLS, class AFetch, class AFin, class WLoad>
__device__ __forceinline__ void tile_gemm(int Kd, AFetch afetch, AFin afin, WLoad wload,
                                          acc_t (&acc)[4][TCOLS / 32], float (*zs)[TR + 4],
                                          float (*ws)[TCOLS + 1], int k_begin = 0, int k_end = -1) {
    if (k_end < 0) k_end = Kd;  // this CTA's slice [k_begin, k_end) of the K loop (split-K)
    constexpr int CJ = TCOLS / 32;  // columns per thread: tx, tx + 32, ...
    constexpr int TK = tk_for<TCOLS>();
    const int tid = threadIdx.x;
    const int ty = tid >> 5, tx = tid & 31;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < CJ; ++j) acc[i][j] = 0;
    constexpr int NA = TR * TK / 256, NW = TCOLS * TK / 256;  // A and W elements per thread per chunk
    float2 ra[NA];
    float rw[NW];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int i = 0; i < NA; ++i) {
            const int e = tid + 256 * i, rr = e / TK, kk = e % TK;
            ra[i] = (k0 + kk < Kd) ? afetch(rr, k0 + kk) : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < NW; ++i) {
            const int e = tid + 256 * i, cc = e / TK, kk = e % TK;
            rw[i] = (k0 + kk < Kd) ? wload(cc, k0 + kk) : 0.f;
        }
    };
    Kd = k_end;  // (bounds below: the slice's end)
    fetch(k_begin);
    for (int k0 = k_begin; k0 < Kd; k0 += TK) {
#pragma unroll
        for (int i = 0; i < NA; ++i) {
            const int e = tid + 256 * i, rr = e / TK, kk = e % TK;
            zs[kk][rr] = (k0 + kk < Kd) ? afin(rr, ra[i]) : 0.f;
        }
#pragma unroll
        for (int i = 0; i < NW; ++i) {
            const int e = tid + 256 * i, cc = e / TK, kk = e % TK;
            ws[kk][cc] = rw[i];
        }
        __syncthreads();
        if (k0 + TK < Kd) fetch(k0 + TK);
#if TBEAM_SIMT_ACC64 == 2
        // fp32 sums of TBEAM_FOLD products, folded into the fp64 accumulators
        #pragma unroll 1
        for (int k8 = 0; k8 < TK; k8 += TBEAM_FOLD) {
            float cacc[4][CJ];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < CJ; ++j) cacc[i][j] = 0.f;
#pragma unroll
            for (int kk = k8; kk < k8 + TBEAM_FOLD; ++kk) {
                const float4 a = *reinterpret_cast<const float4*>(&zs[kk][ty * 4]);
                float b[CJ];
#pragma unroll
                for (int j = 0; j < CJ; ++j) b[j] = ws[kk][tx + 32 * j];
                const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < CJ; ++j) cacc[i][j] = fmaf(av[i], b[j], cacc[i][j]);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < CJ; ++j) acc[i][j] += static_cast<acc_t>(cacc[i][j]);
        }
#else
#pragma unroll 8
        for (int kk = 0; kk < TK; ++kk) {
            const float4 a = *reinterpret_cast<const float4*>(&zs[kk][ty * 4]);
            float b[CJ];
#pragma unroll
            for (int j = 0; j < CJ; ++j) b[j] = ws[kk][tx + 32 * j];
            const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < CJ; ++j)
                    acc[i][j] = fma(static_cast<acc_t>(av[i]), static_cast<acc_t>(b[j]), acc[i][j]);
        }
#endif
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// split-K: the K loop of a tile runs in st.sk_split CTAs (blockIdx.z = slice);
// each stores its fp64 partial tile, the last to arrive (a ticket per tile)
// sums the partials in slice order -- deterministic -- and returns true to run
// the epilogue.  At decode row counts the CUDA-core GEMMs are latency-bound
// on their chain of k-chunks; four slices cut the chain to a quarter.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void splitk_range(int Kd, int TK, int& kb, int& ke) {
    const int KS = gridDim.z, ks = blockIdx.z;
    const int chunks = (Kd + TK - 1) / TK, per = (chunks + KS - 1) / KS;
    kb = min(Kd, ks * per * TK);
    ke = min(Kd, kb + per * TK);
}
template <int CJ>
__device__ bool splitk_reduce(acc_t (&acc)[4][CJ], const DevState& st) {
    const int KS = gridDim.z;
    if (KS == 1) return true;
    __shared__ int s_last;
    const int tid = threadIdx.x;
    const size_t tile = blockIdx.x + static_cast<size_t>(gridDim.x) * blockIdx.y;
    constexpr int PER = 256 * 4 * CJ;
    double* base = st.sk_scratch + tile * KS * PER;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < CJ; ++j) base[blockIdx.z * PER + (i * CJ + j) * 256 + tid] = acc[i][j];
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(st.sk_ticket + tile, 1u) == static_cast<unsigned>(KS - 1);
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < CJ; ++j) {
            double sum = 0.0;
            for (int q = 0; q < KS; ++q) sum += __ldcg(base + q * PER + (i * CJ + j) * 256 + tid);
            acc[i][j] = static_cast<acc_t>(sum);
        }
    if (tid == 0) st.sk_ticket[tile] = 0u;  // ready for the next kernel
    return true;
}

// ---------------------------------------------------------------------------
// encoder projection: encp[b,t,:] = W_enc . enc[b,t,:] + b_enc
// grid (ceil(B*T/32), ceil(J/128))
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) enc_proj_simt(DevModel m, DevState st, int rows) {
    constexpr int TK = tk_for<TC>();
    __shared__ __align__(16) float zs[TK][TR + 4];
    __shared__ float ws[TK][TC + 1];
    const int row0 = blockIdx.x * TR, col0 = blockIdx.y * TC;
    const bool bf = m.prec == 1;
    const float* enc = *st.enc_pp;
    auto afetch = [&](int rr, int k) -> float2 {
        const int row = row0 + rr;
        return make_float2(row < rows ? enc[static_cast<size_t>(row) * m.D + k] : 0.f, 0.f);
    };
    auto afin = [&](int, float2 v) -> float { return bf ? bf16_round(v.x) : v.x; };
    auto wload = [&](int cc, int k) -> float {
        const int col = col0 + cc;
        if (col >= m.J) return 0.f;
        return bf ? __bfloat162float(m.w_enc16[static_cast<size_t>(col) * m.D + k])
                  : m.w_enc[static_cast<size_t>(col) * m.D + k];
    };
    acc_t acc[4][4];
    tile_gemm<TC>(m.D, afetch, afin, wload, acc, zs, ws);
    const int ty = threadIdx.x >> 5, tx = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = row0 + ty * 4 + i;
        if (row >= rows) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int col = col0 + tx + 32 * j;
            if (col < m.J) st.encp[static_cast<size_t>(row) * m.J + col] = acc[i][j] + m.b_enc[col];
        }
    }
}

// ---------------------------------------------------------------------------
// warp top-K over per-lane candidates, order (raw desc, idx asc)
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool beats(float va, int ia, float vb, int ib) {
    return va > vb || (va == vb && ia < ib);
}

// ---------------------------------------------------------------------------
// joint on the compacted active rows of this round.
// grid (ceil(S/32), NT), 256 threads.
// ---------------------------------------------------------------------------
// JC: tile columns (32 -- four times the CTAs of 128 for the latency-bound
// decode shapes -- or 128 when 32-column tiles would exceed the merge bounds)
template <int JC>
__global__ void __launch_bounds__(256) joint_simt(DevModel m, DevLm lm, DevCfg cfg, DevState st, int par) {
    constexpr int TK = tk_for<JC>();
    __shared__ __align__(16) float zs[TK][TR + 4];
    __shared__ float ws[TK][JC + 1];
    __shared__ float os[TR][JC + 1];
    __shared__ int s_slot[TR];
    __shared__ const float* s_enc[TR];
    __shared__ const float* s_pred[TR];
    __shared__ int s_chain[8][kMaxOrder];
    __shared__ float s_acc[8][kMaxOrder];
    __shared__ int s_L[8];

    // (no PDL on the SIMT path: the previous kernel has completed) -- mark
    // whether this round has a decoding stream, for the round statistics
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *st.live = *st.n_done < st.B ? 1 : 0;
    const int count = st.act_count[par];
    const int row0 = blockIdx.x * TR;
    if (row0 >= count) return;
    const int nt = blockIdx.y;
    const int col0 = nt * st.ntile_cols;
    const int ncols = m.R + m.ND;
    const int K = cfg.K;
    const bool bf = m.prec == 1;
    const int tid = threadIdx.x;

    if (tid < TR) {
        const int row = row0 + tid;
        int slot = -1;
        const float* ep = nullptr;
        const float* pp = nullptr;
        if (row < count) {
            slot = st.act_list[par * st.S + row];
            const int b = slot / K;
            const int t = st.t[b];
            ep = st.encp + (static_cast<size_t>(b) * st.Tmax + t) * m.J;
            pp = st.pred + (static_cast<size_t>(b) * st.P + st.pid[slot]) * m.J;
        }
        s_slot[tid] = slot;
        s_enc[tid] = ep;
        s_pred[tid] = pp;
    }
    __syncthreads();

    auto afetch = [&](int rr, int k) -> float2 {
        if (s_slot[rr] < 0) return make_float2(0.f, 0.f);
        return make_float2(s_enc[rr][k], s_pred[rr][k]);
    };
    auto afin = [&](int rr, float2 v) -> float {
        if (s_slot[rr] < 0) return 0.f;
        const float z = tanhf(v.x + v.y);
        return bf ? bf16_round(z) : z;
    };
    auto wload = [&](int cc, int k) -> float {
        const int col = col0 + cc;
        if (col >= ncols || cc >= st.ntile_cols) return 0.f;
        return bf ? __bfloat162float(m.w_out16[static_cast<size_t>(col) * m.J + k])
                  : m.w_out[static_cast<size_t>(col) * m.J + k];
    };
    acc_t acc[4][JC / 32];
    int kb, ke;
    splitk_range(m.J, TK, kb, ke);
    tile_gemm<JC>(m.J, afetch, afin, wload, acc, zs, ws, kb, ke);
    if (!splitk_reduce<JC / 32>(acc, st)) return;

    const int ty = tid >> 5, tx = tid & 31;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < JC / 32; ++j) {
            const int cc = tx + 32 * j;
            const int col = col0 + cc;
            os[ty * 4 + i][cc] = (col < ncols) ? acc[i][j] + m.b_out[col] : 0.f;
        }
    __syncthreads();

    // ---- epilogue: one warp per 4 rows -------------------------------------
    float (*lms)[JC + 1] = ws;  // reuse the W chunk buffer for LM values (TK >= TR rows)
    const int warp = tid >> 5, lane = tid & 31;
    const float lamf = static_cast<float>(cfg.lam);
    const int tile_w = st.ntile_cols;
    for (int q = 0; q < 4; ++q) {
        const int rr = warp * 4 + q;
        const int slot = s_slot[rr];
        if (slot < 0) continue;
        // late-pruning LM row for this tile: unigram level, then higher orders
        // overwrite from shallow to deep (deepest wins, ngram_lm.cpp:379-402)
        if (cfg.late) {
            if (lane == 0) {
                int c = st.lm_state[slot];
                int L = 0;
                double accd = 0.0;
                while (c != 0 && L < kMaxOrder - 1) {
                    s_chain[warp][L] = c;
                    s_acc[warp][L] = static_cast<float>(accd);
                    ++L;
                    accd += lm.backoff[c];
                    c = lm.suffix[c];
                }
                s_chain[warp][L] = 0;
                s_acc[warp][L] = static_cast<float>(accd);
                s_L[warp] = L;
            }
            __syncwarp();
            const int L = s_L[warp];
            const float acc_root = s_acc[warp][L];
            for (int cc = lane; cc < tile_w; cc += 32) {
                const int col = col0 + cc;
                float v = static_cast<float>(kLogZeroFloor);
                if (col < m.V) {
                    const float u = lm.uni[col];
                    if (!isnan(u)) v = fmaxf(acc_root + u, static_cast<float>(kLogZeroFloor));
                    else if (isfinite(lm.unk_prob))
                        v = fmaxf(acc_root + static_cast<float>(lm.unk_prob), static_cast<float>(kLogZeroFloor));
                }
                lms[rr][cc] = v;
            }
            __syncwarp();
            const int hi_tok = min(col0 + tile_w, m.V);
            for (int l = L - 1; l >= 0; --l) {
                const int node = s_chain[warp][l];
                const float al = s_acc[warp][l];
                int lo = lm.cbeg[node], hi = lm.cend[node];
                const int end = hi;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (lm.etok[mid] < col0) lo = mid + 1;
                    else hi = mid;
                }
                for (int e = lo + lane; e < end; e += 32) {
                    const int tk = lm.etok[e];
                    if (tk >= hi_tok) break;
                    const double p = lm.prob[lm.enode[e]];
                    if (!isnan(p)) lms[rr][tk - col0] = fmaxf(al + static_cast<float>(p), static_cast<float>(kLogZeroFloor));
                }
                __syncwarp();
            }
        }
        // log-softmax statistics over the token + blank columns of the tile
        float mx = -INFINITY;
        for (int cc = lane; cc < tile_w; cc += 32) {
            const int col = col0 + cc;
            if (col <= m.V) mx = fmaxf(mx, os[rr][cc]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float sm = 0.f;
        if (mx != -INFINITY)
            for (int cc = lane; cc < tile_w; cc += 32) {
                const int col = col0 + cc;
#if TBEAM_EXACT_EXP
                if (col <= m.V) sm += expf(os[rr][cc] - mx);
#else
                if (col <= m.V) sm += __expf(os[rr][cc] - mx);
#endif
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
        const size_t pb = static_cast<size_t>(slot) * st.NT + nt;
        if (lane == 0) {
            st.part[pb * part_stride(K)] = mx;
            st.part[pb * part_stride(K) + 1] = sm;
        }
        // blank / duration logits
        for (int cc = lane; cc < tile_w; cc += 32) {
            const int col = col0 + cc;
            if (col == m.V) st.blank_logit[slot] = os[rr][cc];
            else if (col > m.V && col < ncols)
                st.dur_logit[static_cast<size_t>(slot) * st.ndx + (col - m.R)] = os[rr][cc];
        }
        // top-K tokens by raw = logit + lambda * lm (late) / logit
        unsigned taken = 0u;
        const int per_lane = (tile_w + 31) / 32;
        for (int i = 0; i < K; ++i) {
            float bv = -INFINITY;
            int bi = 0x7fffffff;
            for (int e = 0; e < per_lane; ++e) {
                const int cc = lane + 32 * e;
                const int col = col0 + cc;
                if (cc >= tile_w || col >= m.V || (taken >> e) & 1u) continue;
                const float raw = cfg.late ? os[rr][cc] + lamf * lms[rr][cc] : os[rr][cc];
                if (beats(raw, col, bv, bi)) {
                    bv = raw;
                    bi = col;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (beats(ov, oi, bv, bi)) {
                    bv = ov;
                    bi = oi;
                }
            }
            if (bi != 0x7fffffff) {
                const int cc = bi - col0;
                if ((cc & 31) == lane) taken |= 1u << (cc >> 5);
            }
            if (lane == 0) {
                float* e = st.part + pb * part_stride(K) + 4 + 4 * i;
                e[0] = bv;
                e[1] = __int_as_float(bi == 0x7fffffff ? -1 : bi);
                e[2] = bi == 0x7fffffff ? 0.f : os[rr][bi - col0];
                e[3] = (bi == 0x7fffffff || !cfg.late) ? 0.f : lms[rr][bi - col0];
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// LSTM step of the token-emitting rows (compacted list upd_list[g&1]):
//   gates = xtab[tok] + W_hh . h[parent];  c' = s(f) c + s(i) tanh(g);
//   h' = s(o) tanh(c')
// Tile columns: 32 hidden units x 4 gates; thread column j = gate j.
// grid (ceil(S/32), ceil(H/32))
// ---------------------------------------------------------------------------
template <int GU>  // hidden units per tile: 8 (4x the CTAs of 32) or 32
__global__ void __launch_bounds__(256) lstm_gates_simt(DevModel m, DevCfg cfg, DevState st, int par) {
    constexpr int GC = 4 * GU;  // tile columns: gate g of unit u at g * GU + u
    constexpr int TK = tk_for<GC>();
    __shared__ __align__(16) float zs[TK][TR + 4];
    __shared__ float ws[TK][GC + 1];
    __shared__ const float* s_h[TR];
    __shared__ int s_slot[TR], s_src[TR], s_dst[TR], s_tok[TR];
    const int cur = par;
    const int count = st.upd_count[cur];
    const int row0 = blockIdx.x * TR;
    if (row0 >= count) return;
    const int u0 = blockIdx.y * GU;
    const int H = m.H;
    const bool bf = m.prec == 1;
    if (threadIdx.x < TR) {
        const int row = row0 + threadIdx.x;
        int slot = -1, src = 0, dst = 0, tok = 0;
        const float* hp = nullptr;
        if (row < count) {
            slot = st.upd_list[cur * st.S + row];
            src = st.upd_src[cur * st.S + row];  // pool rows of parent / child
            dst = st.upd_dst[cur * st.S + row];
            tok = st.upd_tok[cur * st.S + row];
            hp = st.h + static_cast<size_t>(src) * H;
        }
        s_slot[threadIdx.x] = slot;
        s_src[threadIdx.x] = src;
        s_dst[threadIdx.x] = dst;
        s_tok[threadIdx.x] = tok;
        s_h[threadIdx.x] = hp;
    }
    __syncthreads();
    auto afetch = [&](int rr, int k) -> float2 { return make_float2(s_slot[rr] < 0 ? 0.f : s_h[rr][k], 0.f); };
    auto afin = [&](int, float2 v) -> float { return bf ? bf16_round(v.x) : v.x; };
    auto wload = [&](int cc, int k) -> float {
        const int gate = cc / GU, u = u0 + cc % GU;
        if (u >= H) return 0.f;
        const size_t wr = static_cast<size_t>(gate) * H + u;
        return bf ? __bfloat162float(m.w_hh16[wr * H + k]) : m.w_hh[wr * H + k];
    };
    acc_t acc[4][GC / 32];
    int kb, ke;
    splitk_range(H, TK, kb, ke);
    tile_gemm<GC>(H, afetch, afin, wload, acc, zs, ws, kb, ke);
    if (!splitk_reduce<GC / 32>(acc, st)) return;
    const int ty = threadIdx.x >> 5, tx = threadIdx.x & 31;
    // the cell update of (row, unit) needs its four gates in one thread:
    // GU = 32 has them in registers (column tx + 32 g); GU = 8 goes through
    // shared memory (thread = one (row, unit) pair)
    auto cell = [&](int rr, int u, float ai, float af, float ag, float ao) {
        const float* x = m.xtab + static_cast<size_t>(s_tok[rr]) * 4 * H;
        const float gi = ai + x[u];
        const float gf = af + x[H + u];
        const float gg = ag + x[2 * H + u];
        const float go = ao + x[3 * H + u];
        const float ig = 1.f / (1.f + expf(-gi));
        const float fg = 1.f / (1.f + expf(-gf));
        const float og = 1.f / (1.f + expf(-go));
        const float cp = st.c[static_cast<size_t>(s_src[rr]) * H + u];
        const float cn = fg * cp + ig * tanhf(gg);
        st.c[static_cast<size_t>(s_dst[rr]) * H + u] = cn;
        st.h[static_cast<size_t>(s_dst[rr]) * H + u] = og * tanhf(cn);
    };
    if constexpr (GU == 32) {
        const int u = u0 + tx;
        if (u >= H) return;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int rr = ty * 4 + i;
            if (s_slot[rr] < 0) continue;
            cell(rr, u, acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        }
    } else {
        static_assert(GC == 32 && TR * GU == 256, "GU = 8: one (row, unit) pair per thread");
        float (*gs)[TR + 1] = reinterpret_cast<float (*)[TR + 1]>(&zs[0][0]);  // [32 rows][33]: free after the GEMM
#pragma unroll
        for (int i = 0; i < 4; ++i) gs[ty * 4 + i][tx] = acc[i][0];
        __syncthreads();
        const int rr = threadIdx.x / GU, uu = threadIdx.x % GU, u = u0 + uu;
        if (u < H && s_slot[rr] >= 0) cell(rr, u, gs[rr][uu], gs[rr][GU + uu], gs[rr][2 * GU + uu], gs[rr][3 * GU + uu]);
    }
}

// pred[nxt][slot] = W_pred . h'[slot] + b_pred, rows = upd list.
// grid (ceil(S/32), ceil(J/128))
template <int PC>  // tile columns: 32 or 128
__global__ void __launch_bounds__(256) lstm_proj_simt(DevModel m, DevCfg cfg, DevState st, int par) {
    constexpr int TK = tk_for<PC>();
    __shared__ __align__(16) float zs[TK][TR + 4];
    __shared__ float ws[TK][PC + 1];
    __shared__ int s_slot[TR], s_dst[TR];
    const int cur = par;
    const int count = st.upd_count[cur];
    const int row0 = blockIdx.x * TR;
    if (row0 >= count) return;
    const int col0 = blockIdx.y * PC;
    const int H = m.H;
    const bool bf = m.prec == 1;
    if (threadIdx.x < TR) {
        const int row = row0 + threadIdx.x;
        s_slot[threadIdx.x] = row < count ? st.upd_list[cur * st.S + row] : -1;
        s_dst[threadIdx.x] = row < count ? st.upd_dst[cur * st.S + row] : 0;
    }
    __syncthreads();
    auto afetch = [&](int rr, int k) -> float2 {
        return make_float2(s_slot[rr] < 0 ? 0.f : st.h[static_cast<size_t>(s_dst[rr]) * H + k], 0.f);
    };
    auto afin = [&](int, float2 v) -> float { return bf ? bf16_round(v.x) : v.x; };
    auto wload = [&](int cc, int k) -> float {
        const int col = col0 + cc;
        if (col >= m.J) return 0.f;
        return bf ? __bfloat162float(m.w_pred16[static_cast<size_t>(col) * H + k])
                  : m.w_pred[static_cast<size_t>(col) * H + k];
    };
    acc_t acc[4][PC / 32];
    int kb, ke;
    splitk_range(H, TK, kb, ke);
    tile_gemm<PC>(H, afetch, afin, wload, acc, zs, ws, kb, ke);
    if (!splitk_reduce<PC / 32>(acc, st)) return;
    const int ty = threadIdx.x >> 5, tx = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int slot = s_slot[ty * 4 + i];
        if (slot < 0) continue;
        const size_t dst = s_dst[ty * 4 + i];
#pragma unroll
        for (int j = 0; j < PC / 32; ++j) {
            const int col = col0 + tx + 32 * j;
            if (col < m.J) st.pred[dst * m.J + col] = acc[i][j] + m.b_pred[col];
        }
    }
}

// ---- launchers ---------------------------------------------------------------

void launch_enc_proj_simt(const DevModel& m, const DevState& st, int rows, cudaStream_t s) {
    dim3 grid((rows + TR - 1) / TR, (m.J + TC - 1) / TC);
    enc_proj_simt<<<grid, 256, 0, s>>>(m, st, rows);
}

void launch_joint_simt(const DevModel& m, const DevLm& lm, const DevCfg& cfg, const DevState& st, int par,
                       cudaStream_t s) {
    dim3 grid((st.S + TR - 1) / TR, st.NT, st.sk_split);
    if (st.ntile_cols == 32) joint_simt<32><<<grid, 256, 0, s>>>(m, lm, cfg, st, par);
    else joint_simt<TC><<<grid, 256, 0, s>>>(m, lm, cfg, st, par);
}

void launch_lstm_simt(const DevModel& m, const DevCfg& cfg, const DevState& st, int par, cudaStream_t s, int part) {
    dim3 g1((st.S + TR - 1) / TR, (m.H + 7) / 8, st.sk_split);
    if (part != 1) lstm_gates_simt<8><<<g1, 256, 0, s>>>(m, cfg, st, par);
    dim3 g2((st.S + TR - 1) / TR, (m.J + 31) / 32, st.sk_split);
    if (part != 0) lstm_proj_simt<32><<<g2, 256, 0, s>>>(m, cfg, st, par);
}

// joint tile width: 32 columns unless the select's merge bounds (<= 256
// lists, <= 2048 entries per row) need the 128-column tiles
int simt_tile_cols(int ncols, int K) {
    const int nt = (ncols + 31) / 32;
    return nt <= 256 && nt * K <= 2048 ? 32 : TC;
}

}  // namespace tbeam_dev
