// Tensor-core (tcgen05 + TMEM + TMA) GEMMs of the decode, sm_100a, bf16
// operands / fp32 accumulation, each fused with its consumer:
//
//   joint_tc   z[rows] . W_out^T  -> bias, per-tile log-softmax statistics,
//              late-pruning LM fusion, per-row top-K (thread = row)
//              (ToyModel::score_row model.cpp:337-367 + selection_row
//               decoder.cpp:47-61 + the per-row half of prune_topk)
//   gates_tc   h[parent] . W_hh^T -> LSTM cell (i,f,g,o) -> h', c' (+ bf16 h')
//   proj_tc    h' . W_pred^T      -> pred + next round's joint operand
//              z = bf16(tanh(enc_proj + pred))
//   encproj_tc enc . W_enc^T      -> enc_proj (once per decode)
//
// One CTA = one 128 x BN output tile, 4 warps: warp 0 lane 0 issues TMA into a
// 4-stage smem ring, warp 1 lane 0 issues tcgen05.mma (M=128, N=BN, K=16) into
// TMEM and commits each stage back to the producer; then all 4 warps drain
// TMEM with tcgen05.ld (warp w owns TMEM lanes 32w..32w+31 = tile rows) and
// run the fused epilogue.  Row counts are read on device (compacted active /
// token-emitting rows), so one captured graph serves every round.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "device_fns.cuh"
#include "engine.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace tbeam_dev {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int A_BYTES = BM * BK * 2;

// as many K stages as ~200 KB of smem holds: for the decode's K = 640
// (10 k-blocks) narrow tiles keep every load in flight at once
template <int BN>
__host__ __device__ constexpr int tc_stages() {
    return (200 * 1024) / (A_BYTES + BN * BK * 2) > 12 ? 12 : (200 * 1024) / (A_BYTES + BN * BK * 2);
}

template <int BN>
__host__ __device__ constexpr int tc_smem_bytes() {
    return 1024 + tc_stages<BN>() * (A_BYTES + BN * BK * 2) + 256;
}

template <int BN>
__host__ __device__ constexpr uint32_t tmem_cols() {
    return BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
}

// Phase trace of CTA (0,0) of every tc_gemm launch (SM clock): entry,
// prologue done, dependency resolved, accumulator ready, epilogue done.
// Read back with tbeam_debug_gemm_trace (measurement aid, ~free).
__device__ long long g_gemm_trace[32];
__device__ int g_gemm_trace_on;

// ---------------------------------------------------------------------------
// the GEMM skeleton
// ---------------------------------------------------------------------------
template <int BN, class Epi>
__global__ void __launch_bounds__(128, 1)
tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int K,
        int bnv, Epi epi) {
    constexpr int B_BYTES = BN * BK * 2;
    constexpr int STAGES = tc_stages<BN>();
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* done = empty + STAGES;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);

    const int m0 = blockIdx.x * BM;
    const int n0 = blockIdx.y * bnv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool tr = g_gemm_trace_on && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0;
    long long t_entry = 0, t_pro = 0, t_dep = 0, t_acc = 0;
    if (tr) t_entry = clock64();

    // independent prologue, overlapped with the previous kernel's tail (PDL)
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        mbar_fence_init();
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
    }
    if (warp == 0) tmem_alloc(tslot, tmem_cols<BN>());
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    if (tr) t_pro = clock64();
    pdl_trigger();
    pdl_wait();
    if (tr) t_dep = clock64();
    const int rows = epi.rows();
    if (m0 >= rows) {  // no rows for this tile this round
        __syncthreads();
        if (warp == 0) tmem_dealloc(tmem, tmem_cols<BN>());
        return;
    }
    const int nk = (K + BK - 1) / BK;

    if (threadIdx.x == 0) {
        // TMA producer
        const uint32_t bytes = A_BYTES + static_cast<uint32_t>(bnv) * BK * 2;
        for (int kb = 0; kb < nk; ++kb) {
            const int s = kb % STAGES;
            const uint32_t use = kb / STAGES;
            if (kb >= STAGES) mbar_wait(&empty[s], (use & 1u) ^ 1u);
            mbar_expect_tx(&full[s], bytes);
            tma_load_2d(sA + s * A_BYTES, &tmA, &full[s], kb * BK, m0);
            tma_load_2d(sB + s * B_BYTES, &tmB, &full[s], kb * BK, n0);
        }
    } else if (threadIdx.x == 32) {
        // MMA issuer
        const uint32_t idesc = umma_idesc_bf16(BM, bnv);
        for (int kb = 0; kb < nk; ++kb) {
            const int s = kb % STAGES;
            mbar_wait(&full[s], (kb / STAGES) & 1u);
            tc_fence_after();
            const uint32_t a0 = smem_u32(sA + s * A_BYTES);
            const uint32_t b0 = smem_u32(sB + s * B_BYTES);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
                umma_bf16(tmem, umma_desc_sw128(a0 + 32 * k), umma_desc_sw128(b0 + 32 * k), idesc,
                          (kb | k) != 0 ? 1u : 0u);
            umma_commit(&empty[s]);
        }
        umma_commit(done);
    }
    mbar_wait(done, 0);
    __syncwarp();
    tc_fence_after();
    if (tr) t_acc = clock64();
    epi.run(tmem + (static_cast<uint32_t>(warp * 32) << 16), warp, lane, m0, blockIdx.y, n0, bnv, smem);
    if (tr) {
        const long long t_end = clock64();
        long long* g = g_gemm_trace + 8 * Epi::kTrace;
        g[0] += 1;
        g[1] += t_pro - t_entry;
        g[2] += t_dep - t_pro;
        g[3] += t_acc - t_dep;
        g[4] += t_end - t_acc;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, tmem_cols<BN>());
}

// ---------------------------------------------------------------------------
// per-thread top-K (value desc, index asc): unrolled bubble insertion
// ---------------------------------------------------------------------------
template <int KM>
struct TopK {
    float v[KM], lg[KM], lmv[KM];
    int ix[KM];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int q = 0; q < KM; ++q) {
            v[q] = -INFINITY;
            ix[q] = 0x7fffffff;
            lg[q] = 0.f;
            lmv[q] = 0.f;
        }
    }
    // full (value desc, index asc) order, so an element pushed down past an
    // equal value keeps the lower index ahead
    __device__ __forceinline__ void push(float x, int i, float l, float m, int K) {
#pragma unroll
        for (int q = 0; q < KM; ++q) {
            if (q < K && (x > v[q] || (x == v[q] && i < ix[q]))) {
                const float tv = v[q], tl = lg[q], tm = lmv[q];
                const int ti = ix[q];
                v[q] = x;
                ix[q] = i;
                lg[q] = l;
                lmv[q] = m;
                x = tv;
                i = ti;
                l = tl;
                m = tm;
            }
        }
    }
};

// ---------------------------------------------------------------------------
// joint epilogue
// ---------------------------------------------------------------------------
template <int KM>
struct JointEpi {
    static constexpr int kTrace = 0;
    DevModel m;
    DevLm lm;
    DevCfg cfg;
    DevState st;
    int par;
    __device__ int rows() const { return st.act_count[par]; }
    __device__ void run(uint32_t tmem, int warp, int lane, int m0, int nt, int n0, int bnv, uint8_t* scratch) const {
        const int count = st.act_count[par];
        const int r = warp * 32 + lane;
        const int row = m0 + r;
        const bool valid = row < count;
        const int slot = valid ? st.act_list[par * st.S + row] : -1;
        const int ncols = m.R + m.ND;
        const int K = cfg.K;
        const int pitch = bnv + 1;
        float* lmt = reinterpret_cast<float*>(scratch);
        if (cfg.late && valid) {
            // unigram level with <unk> fill, then higher orders overwrite
            // from shallow to deep (ngram_lm.cpp:363-416)
            int chain[kMaxOrder];
            float accs[kMaxOrder];
            int L = 0;
            double accd = 0.0;
            int c = st.lm_state[slot];
            while (c != 0 && L < kMaxOrder) {
                chain[L] = c;
                accs[L] = static_cast<float>(accd);
                ++L;
                accd += lm.backoff[c];
                c = lm.suffix[c];
            }
            const float acc_root = static_cast<float>(accd);
            const float floor_v = static_cast<float>(kLogZeroFloor);
            const float unk = isfinite(lm.unk_prob) ? fmaxf(acc_root + static_cast<float>(lm.unk_prob), floor_v)
                                                    : floor_v;
            for (int cc = 0; cc < bnv; ++cc) {
                const int col = n0 + cc;
                float v = floor_v;
                if (col < m.V) {
                    const float u = lm.uni[col];
                    v = isnan(u) ? unk : fmaxf(acc_root + u, floor_v);
                }
                lmt[r * pitch + cc] = v;
            }
            const int hi_tok = min(n0 + bnv, m.V);
            for (int l = L - 1; l >= 0; --l) {
                const int node = chain[l];
                int lo = lm.cbeg[node], hi = lm.cend[node];
                const int end = hi;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (lm.etok[mid] < n0) lo = mid + 1;
                    else hi = mid;
                }
                for (int e = lo; e < end; ++e) {
                    const int tk = lm.etok[e];
                    if (tk >= hi_tok) break;
                    const double p = lm.prob[lm.enode[e]];
                    if (!isnan(p)) lmt[r * pitch + (tk - n0)] = fmaxf(accs[l] + static_cast<float>(p), floor_v);
                }
            }
        }
        const float lamf = static_cast<float>(cfg.lam);
        float mx = -INFINITY, sm = 0.f;
        TopK<KM> top;
        top.init();
        // this tile's bias, staged once (per-element global loads serialise)
        float* bias = reinterpret_cast<float*>(scratch + 190 * 1024);
        for (int c = r; c < bnv; c += 128) bias[c] = n0 + c < ncols ? m.b_out[n0 + c] : 0.f;
        __syncthreads();
        for (int c0 = 0; c0 < bnv; c0 += 32) {
            float v[32];
            tmem_ld32(tmem + c0, v);
            if (!valid) continue;
            const int lim = min(32, min(bnv, ncols - n0) - c0);  // columns of this chunk
            // logits (bias added) and the chunk max over token + blank columns
            float cmax = -INFINITY;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                v[j] = j < lim ? v[j] + bias[c0 + j] : -INFINITY;
                if (n0 + c0 + j <= m.V) cmax = fmaxf(cmax, v[j]);
            }
            // online log-sum-exp, one rescale per chunk
            if (cmax > -INFINITY) {
                const float nm = fmaxf(mx, cmax);
                float acc = sm * __expf(mx - nm);
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (n0 + c0 + j <= m.V) acc += __expf(v[j] - nm);
                sm = acc;
                mx = nm;
            }
            // token columns -> per-row top-K; blank / duration columns stored
            const int ntok = min(lim, m.V - (n0 + c0));
            if constexpr (KM <= 8) {
                // fully unrolled so v[] stays in registers
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if (j < ntok) {
                        const float lv = cfg.late ? lmt[r * pitch + c0 + j] : 0.f;
                        const float raw = cfg.late ? v[j] + lamf * lv : v[j];
                        if (raw > top.v[KM - 1] || K < KM) top.push(raw, n0 + c0 + j, v[j], lv, K);
                    } else if (j < lim) {
                        const int col = n0 + c0 + j;
                        if (col == m.V) st.blank_logit[slot] = v[j];
                        else st.dur_logit[static_cast<size_t>(slot) * st.ndx + (col - m.R)] = v[j];
                    }
                }
            } else {
                // wide beams: stage the chunk in smem (a 32-entry push unrolled
                // 32 times would not fit the register file)
                float* vb = reinterpret_cast<float*>(scratch + 132 * 1024) + r * 33;
#pragma unroll
                for (int j = 0; j < 32; ++j) vb[j] = v[j];
#pragma unroll 1
                for (int j = 0; j < lim; ++j) {
                    const float x = vb[j];
                    if (j < ntok) {
                        const float lv = cfg.late ? lmt[r * pitch + c0 + j] : 0.f;
                        const float raw = cfg.late ? x + lamf * lv : x;
                        if (raw > top.v[KM - 1] || K < KM) top.push(raw, n0 + c0 + j, x, lv, K);
                    } else {
                        const int col = n0 + c0 + j;
                        if (col == m.V) st.blank_logit[slot] = x;
                        else st.dur_logit[static_cast<size_t>(slot) * st.ndx + (col - m.R)] = x;
                    }
                }
            }
        }
        if (!valid) return;
        const size_t pb = static_cast<size_t>(slot) * st.NT + nt;
        st.pmax[pb] = mx;
        st.psum[pb] = sm;
#pragma unroll
        for (int q = 0; q < KM; ++q) {
            if (q >= K) break;
            const size_t o = pb * K + q;
            const bool ok = top.ix[q] != 0x7fffffff;
            st.ptop_raw[o] = top.v[q];
            st.ptop_idx[o] = ok ? top.ix[q] : -1;
            st.ptop_logit[o] = top.lg[q];
            st.ptop_lm[o] = top.lmv[q];
        }
    }
};

// ---------------------------------------------------------------------------
// encoder projection epilogue: encp = acc + b_enc
// ---------------------------------------------------------------------------
struct EncProjEpi {
    static constexpr int kTrace = 3;
    DevModel m;
    DevState st;
    int nrows;
    __device__ int rows() const { return nrows; }
    __device__ void run(uint32_t tmem, int warp, int lane, int m0, int nt, int n0, int bnv, uint8_t*) const {
        const int row = m0 + warp * 32 + lane;
        const bool valid = row < nrows;
        float* out = st.encp + static_cast<size_t>(row) * m.J;
        for (int c0 = 0; c0 < bnv; c0 += 32) {
            float v[32];
            tmem_ld32(tmem + c0, v);
            if (!valid) continue;
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
                const int col = n0 + c0 + j;
                if (c0 + j >= bnv || col >= m.J) break;
                if (col + 3 < m.J && c0 + j + 3 < bnv) {
                    float4 q = make_float4(v[j] + m.b_enc[col], v[j + 1] + m.b_enc[col + 1],
                                           v[j + 2] + m.b_enc[col + 2], v[j + 3] + m.b_enc[col + 3]);
                    *reinterpret_cast<float4*>(out + col) = q;
                } else {
                    for (int q = 0; q < 4 && col + q < m.J && c0 + j + q < bnv; ++q)
                        out[col + q] = v[j + q] + m.b_enc[col + q];
                }
            }
        }
    }
};

// ---------------------------------------------------------------------------
// LSTM gates epilogue: tile nt = hidden units [32nt, 32nt+32) x (i,f,g,o)
// ---------------------------------------------------------------------------
struct GatesEpi {
    static constexpr int kTrace = 1;
    DevModel m;
    DevState st;
    int par;
    __device__ int rows() const { return st.upd_count[par]; }
    __device__ void run(uint32_t tmem, int warp, int lane, int m0, int nt, int n0, int bnv, uint8_t*) const {
        const int cur = par, nxt = par ^ 1;
        const int count = st.upd_count[cur];
        const int row = m0 + warp * 32 + lane;
        const bool valid = row < count;
        float gi[32], gf[32], gg[32], go[32];
        tmem_ld32(tmem + 0, gi);
        tmem_ld32(tmem + 32, gf);
        tmem_ld32(tmem + 64, gg);
        tmem_ld32(tmem + 96, go);
        if (!valid) return;
        const size_t S = st.S;
        const int H = m.H;
        const int slot = st.upd_list[cur * S + row];
        const int parent = st.sel_parent[slot];
        const int tok = st.sel_token[slot];
        const int u0 = nt * 32;
        const float* __restrict__ x = m.xtab + static_cast<size_t>(tok) * 4 * H + u0;
        const float4* __restrict__ cp = reinterpret_cast<const float4*>(st.c + (cur * S + parent) * H + u0);
        float4* __restrict__ cn = reinterpret_cast<float4*>(st.c + (nxt * S + slot) * H + u0);
        float4* __restrict__ hn = reinterpret_cast<float4*>(st.h + (nxt * S + slot) * H + u0);
        uint4* __restrict__ hb = reinterpret_cast<uint4*>(st.hB16 + static_cast<size_t>(row) * st.Hp + u0);
        // all loads of this thread's 32 units issued up front (c and the gate inputs)
        float4 cpv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) cpv[q] = cp[q];
#pragma unroll
        for (int q = 0; q < 8; ++q) {  // 4 hidden units per step, all loads vectorised
            const float4 xi = __ldg(reinterpret_cast<const float4*>(x) + q);
            const float4 xf = __ldg(reinterpret_cast<const float4*>(x + H) + q);
            const float4 xg = __ldg(reinterpret_cast<const float4*>(x + 2 * H) + q);
            const float4 xo = __ldg(reinterpret_cast<const float4*>(x + 3 * H) + q);
            const float4 c4 = cpv[q];
            const float xa[4][4] = {{xi.x, xi.y, xi.z, xi.w}, {xf.x, xf.y, xf.z, xf.w},
                                    {xg.x, xg.y, xg.z, xg.w}, {xo.x, xo.y, xo.z, xo.w}};
            const float ca[4] = {c4.x, c4.y, c4.z, c4.w};
            float cn4[4], hn4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int u = q * 4 + e;
                const float ig = __fdividef(1.f, 1.f + __expf(-(gi[u] + xa[0][e])));
                const float fg = __fdividef(1.f, 1.f + __expf(-(gf[u] + xa[1][e])));
                const float g = tanhf(gg[u] + xa[2][e]);
                const float og = __fdividef(1.f, 1.f + __expf(-(go[u] + xa[3][e])));
                cn4[e] = fg * ca[e] + ig * g;
                hn4[e] = og * tanhf(cn4[e]);
            }
            cn[q] = make_float4(cn4[0], cn4[1], cn4[2], cn4[3]);
            hn[q] = make_float4(hn4[0], hn4[1], hn4[2], hn4[3]);
            const __nv_bfloat162 h01 = __floats2bfloat162_rn(hn4[0], hn4[1]);
            const __nv_bfloat162 h23 = __floats2bfloat162_rn(hn4[2], hn4[3]);
            uint2 pk;
            pk.x = *reinterpret_cast<const uint32_t*>(&h01);
            pk.y = *reinterpret_cast<const uint32_t*>(&h23);
            reinterpret_cast<uint2*>(hb)[q] = pk;
        }
    }
};

// ---------------------------------------------------------------------------
// prediction projection epilogue: pred = acc + b_pred; next round's z row
// ---------------------------------------------------------------------------
struct ProjEpi {
    static constexpr int kTrace = 2;
    DevModel m;
    DevState st;
    int par;
    __device__ int rows() const { return st.upd_count[par]; }
    __device__ void run(uint32_t tmem, int warp, int lane, int m0, int nt, int n0, int bnv, uint8_t*) const {
        const int cur = par, nxt = par ^ 1;
        const int count = st.upd_count[cur];
        const int row = m0 + warp * 32 + lane;
        const bool valid = row < count;
        const size_t S = st.S;
        int slot = 0, pos = -1;
        const float* ep = nullptr;
        if (valid) {
            slot = st.upd_list[cur * S + row];
            pos = st.act_pos[slot];
            const int b = slot / st.K;
            ep = st.encp + (static_cast<size_t>(b) * st.Tmax + min(st.t[b], st.Tmax - 1)) * m.J;
        }
        float* pd = st.pred + (nxt * S + slot) * m.J;
        for (int c0 = 0; c0 < bnv; c0 += 32) {
            float v[32];
            tmem_ld32(tmem + c0, v);
            const int col0 = n0 + c0;
            if (!valid || col0 >= m.J) continue;
            if (col0 + 32 <= m.J) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float4 bq = __ldg(reinterpret_cast<const float4*>(m.b_pred + col0) + q);
                    const float4 p = make_float4(v[4 * q] + bq.x, v[4 * q + 1] + bq.y, v[4 * q + 2] + bq.z,
                                                 v[4 * q + 3] + bq.w);
                    reinterpret_cast<float4*>(pd + col0)[q] = p;
                    if (pos >= 0) {
                        const float4 e = reinterpret_cast<const float4*>(ep + col0)[q];
                        const __nv_bfloat162 z01 = __floats2bfloat162_rn(tanhf(e.x + p.x), tanhf(e.y + p.y));
                        const __nv_bfloat162 z23 = __floats2bfloat162_rn(tanhf(e.z + p.z), tanhf(e.w + p.w));
                        uint2 pk;
                        pk.x = *reinterpret_cast<const uint32_t*>(&z01);
                        pk.y = *reinterpret_cast<const uint32_t*>(&z23);
                        reinterpret_cast<uint2*>(st.z16 + static_cast<size_t>(pos) * st.Jp + col0)[q] = pk;
                    }
                }
            } else {
                for (int j = 0; j < 32 && col0 + j < m.J; ++j) {
                    const float p = v[j] + m.b_pred[col0 + j];
                    pd[col0 + j] = p;
                    if (pos >= 0)
                        st.z16[static_cast<size_t>(pos) * st.Jp + col0 + j] =
                            __float2bfloat16_rn(tanhf(ep[col0 + j] + p));
                }
            }
        }
    }
};

// ---------------------------------------------------------------------------
// host side: tensor maps + launchers
// ---------------------------------------------------------------------------
namespace {

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

void load_encode() {
    if (g_encode) return;
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
        throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

template <int BN, class Epi>
void launch_gemm(const TcMap& a, const TcMap& b, int K, int bnv, int m_tiles, int n_tiles, const Epi& epi,
                 cudaStream_t s) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(m_tiles, n_tiles);
    lc.blockDim = dim3(128);
    lc.dynamicSmemBytes = tc_smem_bytes<BN>();
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    cudaLaunchKernelEx(&lc, tc_gemm<BN, Epi>, a.map, b.map, K, bnv, epi);
}

template <int BN, class Epi>
void set_smem_attr() {
    cudaFuncSetAttribute(tc_gemm<BN, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem_bytes<BN>());
}

}  // namespace

TcMap make_tc_map(const void* base, int rows, int k, int pitch_elems, int box_rows) {
    load_encode();
    TcMap t{};
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch_elems) * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t es[2] = {1, 1};
    const CUresult r = g_encode(&t.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                                box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return t;
}

void gemm_trace(int enable, long long* out) {
    if (out) {
        cudaMemcpyFromSymbol(out, g_gemm_trace, sizeof(long long) * 32);
    }
    long long z[32] = {};
    cudaMemcpyToSymbol(g_gemm_trace, z, sizeof(z));
    cudaMemcpyToSymbol(g_gemm_trace_on, &enable, sizeof(int));
}

void configure_tc_kernels() {
    set_smem_attr<32, JointEpi<1>>();
    set_smem_attr<32, JointEpi<4>>();
    set_smem_attr<32, JointEpi<8>>();
    set_smem_attr<32, JointEpi<16>>();
    set_smem_attr<32, JointEpi<32>>();
    set_smem_attr<64, JointEpi<1>>();
    set_smem_attr<64, JointEpi<4>>();
    set_smem_attr<64, JointEpi<8>>();
    set_smem_attr<64, JointEpi<16>>();
    set_smem_attr<64, JointEpi<32>>();
    set_smem_attr<256, JointEpi<1>>();
    set_smem_attr<256, JointEpi<4>>();
    set_smem_attr<256, JointEpi<8>>();
    set_smem_attr<256, JointEpi<16>>();
    set_smem_attr<256, JointEpi<32>>();
    set_smem_attr<128, EncProjEpi>();
    set_smem_attr<128, GatesEpi>();
    set_smem_attr<32, ProjEpi>();
}

void launch_joint_tc(const DevModel& m, const DevLm& lm, const DevCfg& cfg, const DevState& st, const TcPlan& p,
                     int par, cudaStream_t s) {
    const int m_tiles = (st.S + BM - 1) / BM;
    const int K = cfg.K;
#define TBEAM_JOINT(BNV, KMV)                                                                         \
    launch_gemm<BNV, JointEpi<KMV>>(p.z, p.wout, m.J, p.joint_bnv, m_tiles, st.NT,                  \
                                    JointEpi<KMV>{m, lm, cfg, st, par}, s)
    if (p.joint_bn == 32) {
        if (K <= 1) TBEAM_JOINT(32, 1);
        else if (K <= 4) TBEAM_JOINT(32, 4);
        else if (K <= 8) TBEAM_JOINT(32, 8);
        else if (K <= 16) TBEAM_JOINT(32, 16);
        else TBEAM_JOINT(32, 32);
    } else if (p.joint_bn == 64) {
        if (K <= 1) TBEAM_JOINT(64, 1);
        else if (K <= 4) TBEAM_JOINT(64, 4);
        else if (K <= 8) TBEAM_JOINT(64, 8);
        else if (K <= 16) TBEAM_JOINT(64, 16);
        else TBEAM_JOINT(64, 32);
    } else {
        if (K <= 1) TBEAM_JOINT(256, 1);
        else if (K <= 4) TBEAM_JOINT(256, 4);
        else if (K <= 8) TBEAM_JOINT(256, 8);
        else if (K <= 16) TBEAM_JOINT(256, 16);
        else TBEAM_JOINT(256, 32);
    }
#undef TBEAM_JOINT
}

void launch_encproj_tc(const DevModel& m, const DevState& st, const TcPlan& p, int rows, cudaStream_t s) {
    const int m_tiles = (rows + BM - 1) / BM;
    const int n_tiles = (m.J + 127) / 128;
    launch_gemm<128, EncProjEpi>(p.enc, p.wenc, m.D, 128, m_tiles, n_tiles, EncProjEpi{m, st, rows}, s);
}

void launch_lstm_tc(const DevModel& m, const DevState& st, const TcPlan& p, int par, cudaStream_t s) {
    const int m_tiles = (st.S + BM - 1) / BM;
    launch_gemm<128, GatesEpi>(p.hA, p.whh, m.H, 128, m_tiles, m.H / 32, GatesEpi{m, st, par}, s);
    launch_gemm<32, ProjEpi>(p.hB, p.wpred, m.H, 32, m_tiles, (m.J + 31) / 32, ProjEpi{m, st, par}, s);
}

}  // namespace tbeam_dev
