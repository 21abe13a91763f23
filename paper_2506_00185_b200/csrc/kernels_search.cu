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
#include <cstdint>

#include "device_fns.cuh"
#include "engine.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace tbeam_dev {

namespace {

struct SelSmem {
    // byte offsets of every array in the dynamic shared buffer
    size_t sc, lse, asrb, fbl, l1m, dlp, tkv, csc, nsc, edon, cidx, hs, ln, ls, fr, tn, lmst,
        act, tkn, tki, tkw, ck, cdi, cdest, sel, ea, ec, don, sraw, sidx, total;
    // nstage = per-warp staging entries (NT*K of the joint partials), nw = warps
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
        sraw = take(4 * static_cast<size_t>(nstage) * nw);
        sidx = take(4 * static_cast<size_t>(nstage) * nw);
        total = o;
    }
};

__device__ __forceinline__ bool beats_f(float va, int ia, float vb, int ib) {
    return va > vb || (va == vb && ia < ib);
}

}  // namespace

int select_threads(int K) { return K <= 8 ? 128 : 256; }
size_t select_smem_bytes(int K, int ND, int NT) {
    return SelSmem(K, ND > 0 ? ND : 1, NT * K, select_threads(K) / 32).total;
}

// phase trace of select CTA 0 (SM clock), measurement aid
__device__ long long g_sel_trace[8];
__device__ int g_sel_trace_on;
#define SEL_MARK(k)                                                                      \
    do {                                                                                 \
        if (g_sel_trace_on && blockIdx.x == 0 && threadIdx.x == 0) {                      \
            const long long _t = clock64();                                              \
            g_sel_trace[k] += _t - sel_t0;                                               \
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
            st.z16[static_cast<size_t>(b) * st.Jp + j] = __float2bfloat16_rn(tanhf(ep[j] + pp[j]));
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
// select: one CTA (256 threads) per stream
// ---------------------------------------------------------------------------
__device__ __forceinline__ void select_stream(const DevModel& m, const DevLm& lm, const DevCfg& cfg,
                                           const DevState& st, const int par) {
    const int b = blockIdx.x;
    extern __shared__ __align__(16) unsigned char smem[];
    const int K = cfg.K, V = m.V, R = m.R, ND = m.ND, ndx = st.ndx, RS = K + ndx;
    const SelSmem L(K, ndx, st.NT * K, blockDim.x >> 5);
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
    int* tkw = reinterpret_cast<int*>(smem + L.tkw);
    float* sraw = reinterpret_cast<float*>(smem + L.sraw);
    int* sidx = reinterpret_cast<int*>(smem + L.sidx);
    __shared__ int n_edges, n_final, n_active, n_early;
    __shared__ int s_par[kMaxBeam], s_tok[kMaxBeam], s_upos[kMaxBeam], s_apos[kMaxBeam];
    __shared__ int s_pid[kMaxBeam], s_npid[kMaxBeam];  // prediction-state pool entries (old / new)

    const int tid = threadIdx.x, nthr = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31, nwarps = nthr >> 5;
    long long sel_t0 = clock64();
    const int cur = par, nxt = par ^ 1;
    const int col = st.col[b];  // this stream's trie column (= its round count)
    const int t = st.t[b], r = st.r[b], T = st.T[b];
    const bool last_round = r == cfg.token_rounds;
    const size_t S = st.S;

    // 1. slot state ------------------------------------------------------------
    if (tid < K) {
        const int s = b * K + tid;
        sc[tid] = st.score[s];
        ln[tid] = st.len[s];
        hs[tid] = st.hash[s];
        ls[tid] = st.last[s];
        fr[tid] = st.f[s];
        tn[tid] = st.tnode[s];
        lmst[tid] = st.lm_state[s];
        act[tid] = (sc[tid] != -INFINITY && fr[tid] == t) ? 1 : 0;
        don[tid] = cfg.quirk ? st.sdonated[s] : 0;
        tkn[tid] = 0;
        s_pid[tid] = st.pid[s];
    }
    if (tid == 0) {
        n_edges = 0;
        n_final = 0;
        n_early = 0;
    }
    __syncthreads();

    // 2. combine the joint's tile partials, one warp per active slot -----------
    const int NT = st.NT;
    const int nent = NT * K;
    for (int i = warp; i < K; i += nwarps) {
        if (!act[i]) continue;
        const size_t s = static_cast<size_t>(b) * K + i;
        float mx = -INFINITY;
        const int ps = part_stride(K);
        const float* rec = st.part + s * NT * ps;
        for (int q = lane; q < NT; q += 32) mx = fmaxf(mx, rec[q * ps]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        double sum = 0.0;
        for (int q = lane; q < NT; q += 32) {
            const float pm = rec[q * ps];
            if (pm != -INFINITY) sum += static_cast<double>(rec[q * ps + 1]) * exp(static_cast<double>(pm) - mx);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        const double lz = static_cast<double>(mx) + log(sum);
        const double ab = static_cast<double>(st.blank_logit[s]) - lz;
        const double l1 = (cfg.late && cfg.blank_mode == 1) ? d_log1mexp(ab) : 0.0;
        // durations (TDT): own log-softmax
        if (ND > 0) {
            const float dv = lane < ND ? st.dur_logit[s * ndx + lane] : -INFINITY;
            float dm = dv;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dm = fmaxf(dm, __shfl_xor_sync(0xffffffffu, dm, o));
            double de = lane < ND ? exp(static_cast<double>(dv) - dm) : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) de += __shfl_xor_sync(0xffffffffu, de, o);
            if (lane < ND) dlp[i * ndx + lane] = static_cast<double>(dv) - (static_cast<double>(dm) + log(de));
        }
        // top-K tokens: K-way merge of the NT per-tile lists (each sorted by
        // raw desc, idx asc), staged in smem with one coalesced pass; lane
        // owns tiles lane, lane+32, ... (NT <= 256)
        float* wr = sraw + static_cast<size_t>(warp) * nent;
        int* wi_ = sidx + static_cast<size_t>(warp) * nent;
        for (int e = lane; e < nent; e += 32) {
            const int q = e / K, pos = e - q * K;
            const float2 ri = *reinterpret_cast<const float2*>(rec + q * ps + 4 + 4 * pos);
            wr[e] = ri.x;
            wi_[e] = __float_as_int(ri.y);
        }
        __syncwarp();
        float hv[8];
        int hi[8], hp[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int q = lane + 32 * u;
            hv[u] = -INFINITY;
            hi[u] = 0x7fffffff;
            hp[u] = 0;
            if (q < NT && wi_[q * K] >= 0) {
                hv[u] = wr[q * K];
                hi[u] = wi_[q * K];
            }
        }
        int found = 0;
        for (int j = 0; j < K; ++j) {
            float bv = -INFINITY;
            int bi = 0x7fffffff, bu = -1;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (hi[u] != 0x7fffffff && beats_f(hv[u], hi[u], bv, bi)) {
                    bv = hv[u];
                    bi = hi[u];
                    bu = u;
                }
            float wv = bv;
            int wi = bi;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, wv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, wi, o);
                if (beats_f(ov, oi, wv, wi)) {
                    wv = ov;
                    wi = oi;
                }
            }
            if (wi == 0x7fffffff) break;
            if (bu >= 0 && bi == wi) {  // this lane holds the winner (column ids are unique)
                int q = 0, pos = 0;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (u == bu) {
                        q = lane + 32 * u;
                        pos = hp[u];
                    }
                tkw[i * K + j] = q * K + pos;  // entry of the winner in this row's list
                tki[i * K + j] = wi;
                const int np = pos + 1;
                float nv = -INFINITY;
                int ni = 0x7fffffff;
                if (np < K && wi_[q * K + np] >= 0) {
                    nv = wr[q * K + np];
                    ni = wi_[q * K + np];
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (u == bu) {
                        hv[u] = nv;
                        hi[u] = ni;
                        hp[u] = np;
                    }
            }
            ++found;
        }
        __syncwarp();
        // fused values of the winners: their logits / LM values in one pass
        if (lane < found) {
            const int e = tkw[i * K + lane];
            const int q = e / K, pos = e - q * K;
            const float2 ll = *reinterpret_cast<const float2*>(rec + q * ps + 4 + 4 * pos + 2);
            const double lmv = cfg.late ? static_cast<double>(ll.y) : 0.0;
            tkv[i * K + lane] = fused_token(cfg, static_cast<double>(ll.x), lz, lmv, l1);
        }
        if (lane == 0) {
            tkn[i] = found;
            lse[i] = lz;
            asrb[i] = ab;
            fbl[i] = fused_blank(cfg, ab);
            l1m[i] = l1;
        }
    }
    __syncthreads();

    SEL_MARK(1);
    // 3. AES++ maximum-length prefix combination (round 0 of a frame) ------------
    const bool do_prefix = cfg.algo == 2 && cfg.prefix && r == 0 && (ND == 0 || m.di0 >= 0);
    if (do_prefix) {
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
        const int ne = n_edges;
        if (tid == 0) {  // sort by (len(receiver), receiver, donor)
            for (int x = 1; x < ne; ++x) {
                const int a = ea[x], c = ec[x];
                int y = x - 1;
                while (y >= 0) {
                    const int ya = ea[y], yc = ec[y];
                    const bool gt = ln[yc] > ln[c] || (ln[yc] == ln[c] && (yc > c || (yc == c && ya > a)));
                    if (!gt) break;
                    ea[y + 1] = ya;
                    ec[y + 1] = yc;
                    --y;
                }
                ea[y + 1] = a;
                ec[y + 1] = c;
            }
        }
        __syncthreads();
        // donor's fused value of the receiver's last token: z_a . W_out[last] + b
        for (int e = warp; e < ne; e += nwarps) {
            const int a = ea[e], c = ec[e];
            const int k = ls[c];
            const size_t sa = static_cast<size_t>(b) * K + a;
            const float* ep = st.encp + (static_cast<size_t>(b) * st.Tmax + t) * m.J;
            const float* pp = st.pred + (static_cast<size_t>(b) * st.P + s_pid[a]) * m.J;
            float acc = 0.f;
            for (int j = lane; j < m.J; j += 32) {
                float z = tanhf(ep[j] + pp[j]);
                float w;
                if (m.prec == 1) {
                    z = bf16_round(z);
                    w = __bfloat162float(m.w_out16[static_cast<size_t>(k) * m.J + j]);
                } else {
                    w = m.w_out[static_cast<size_t>(k) * m.J + j];
                }
                acc = fmaf(z, w, acc);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) {
                const double logit = static_cast<double>(acc + m.b_out[k]);
                const double lmv = cfg.late ? lm_vocab_value(lm, lmst[a], k) : 0.0;
                double part = fused_token(cfg, logit, lse[a], lmv, l1m[a]);
                if (ND > 0) part += dlp[a * ndx + m.di0];
                if (cfg.early) {
                    double term = lm_score_token(lm, lmst[a], k);
                    if (cfg.blank_mode == 1) term += d_log1mexp(asrb[a]);
                    part += cfg.lam * term;
                }
                edon[e] = part;
            }
        }
        __syncthreads();
        if (tid == 0) {  // serial application in sorted order
            for (int e = 0; e < ne; ++e) {
                const int a = ea[e], c = ec[e];
                sc[c] = d_merge(sc[c], sc[a] + edon[e], cfg.merge_mode);
                don[a] = 1;
            }
            if (cfg.early) n_early += ne;
        }
        __syncthreads();
    }

    SEL_MARK(2);
    // 4. candidates, slot-major regions of RS entries ---------------------------
    for (int x = tid; x < K * RS; x += nthr) {
        csc[x] = -INFINITY;
        ck[x] = -1;
    }
    __syncthreads();
    for (int i = tid; i < K; i += nthr) {
        if (sc[i] == -INFINITY) continue;
        const double base = sc[i];
        const long long sb = static_cast<long long>(i) * R * ndx;
        const int rb = i * RS;
        if (fr[i] != t) {  // complete: carry the slot with its blank column
            csc[rb + K] = base;
            cidx[rb + K] = sb + static_cast<long long>(V) * ndx;
            ck[rb + K] = V;
            cdi[rb + K] = 0;
            cdest[rb + K] = fr[i];
            continue;
        }
        const bool allow = !don[i] && ln[i] < cfg.max_len;
        if (ND == 0) {
            if (allow && !last_round)
                for (int j = 0; j < tkn[i]; ++j) {
                    csc[rb + j] = tkv[i * K + j] + base;
                    cidx[rb + j] = sb + tki[i * K + j];
                    ck[rb + j] = tki[i * K + j];
                    cdi[rb + j] = 0;
                    cdest[rb + j] = t;
                }
            csc[rb + K] = base + fbl[i];
            cidx[rb + K] = sb + V;
            ck[rb + K] = V;
            cdi[rb + K] = 0;
            cdest[rb + K] = min(t + 1, T);
        } else {
            if (allow) {
                // top-K (token, duration) combos of this slot; insertion select
                int nsel = 0;
                for (int j = 0; j < tkn[i]; ++j) {
                    const int k = tki[i * K + j];
                    for (int d = 0; d < ND; ++d) {
                        const int dv = m.durations[d];
                        if (last_round && dv == 0) continue;
                        const double v = tkv[i * K + j] + dlp[i * ndx + d];
                        const long long id = sb + static_cast<long long>(k) * ndx + d;
                        if (nsel < K) {
                            csc[rb + nsel] = v;
                            cidx[rb + nsel] = id;
                            ck[rb + nsel] = k;
                            cdi[rb + nsel] = d;
                            ++nsel;
                        } else {
                            int worst = 0;
                            for (int q = 1; q < K; ++q) {
                                const bool qw = csc[rb + q] < csc[rb + worst] ||
                                                (csc[rb + q] == csc[rb + worst] && cidx[rb + q] > cidx[rb + worst]);
                                if (qw) worst = q;
                            }
                            const bool better = v > csc[rb + worst] || (v == csc[rb + worst] && id < cidx[rb + worst]);
                            if (better) {
                                csc[rb + worst] = v;
                                cidx[rb + worst] = id;
                                ck[rb + worst] = k;
                                cdi[rb + worst] = d;
                            }
                        }
                    }
                }
                for (int q = 0; q < nsel; ++q) {
                    csc[rb + q] = base + csc[rb + q];
                    cdest[rb + q] = min(t + m.durations[cdi[rb + q]], T);
                }
            }
            for (int d = 0; d < ND; ++d) {
                const int dv = m.durations[d];
                if (dv < 1) continue;  // blank must advance
                csc[rb + K + d] = base + (fbl[i] + dlp[i * ndx + d]);
                cidx[rb + K + d] = sb + static_cast<long long>(V) * ndx + d;
                ck[rb + K + d] = V;
                cdi[rb + K + d] = d;
                cdest[rb + K + d] = min(t + dv, T);
            }
        }
    }
    __syncthreads();

    // 5. recombination of the frame-leaving blank column by (HypKey, dest) -------
    const int nb = K * ndx;
    for (int x = tid; x < nb; x += nthr) {
        const int i = x / ndx, e = i * RS + K + (x % ndx);
        nsc[x] = csc[e];
        if (csc[e] == -INFINITY) continue;
        bool leader = true;
        for (int y = 0; y < x && leader; ++y) {
            const int iy = y / ndx, ey = iy * RS + K + (y % ndx);
            if (csc[ey] != -INFINITY && hs[iy] == hs[i] && ln[iy] == ln[i] && ls[iy] == ls[i] &&
                cdest[ey] == cdest[e])
                leader = false;
        }
        if (!leader) {
            nsc[x] = -INFINITY;
            continue;
        }
        double accv = csc[e];
        for (int y = x + 1; y < nb; ++y) {
            const int iy = y / ndx, ey = iy * RS + K + (y % ndx);
            if (csc[ey] != -INFINITY && hs[iy] == hs[i] && ln[iy] == ln[i] && ls[iy] == ls[i] &&
                cdest[ey] == cdest[e])
                accv = d_merge(accv, csc[ey], cfg.merge_mode);
        }
        nsc[x] = accv;
    }
    __syncthreads();
    for (int x = tid; x < nb; x += nthr) {
        const int i = x / ndx;
        csc[i * RS + K + (x % ndx)] = nsc[x];
    }
    __syncthreads();

    // 6. prune_topk: rank by (score desc, index asc) -----------------------------
    const int total = K * RS;
    for (int x = tid; x < total; x += nthr) {
        const double v = csc[x];
        if (v == -INFINITY) continue;
        atomicAdd(&n_final, 1);
        const long long id = cidx[x];
        int rank = 0;
        for (int y = 0; y < total && rank < K; ++y) {
            const double w = csc[y];
            if (w == -INFINITY) continue;
            if (w > v || (w == v && cidx[y] < id)) ++rank;
        }
        if (rank < K) sel[rank] = x;
    }
    __syncthreads();

    SEL_MARK(3);
    // 7. expansion ---------------------------------------------------------------
    const int F = min(n_final, K);
    double n_score = -INFINITY;
    int n_len = 0, n_last = -1, n_f = T, n_tn = -1, n_lm = 0, n_par = 0, n_tok = -1;
    unsigned long long n_hash = 0ull;
    if (tid < K) {
        const int j = tid;
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
                if (cfg.early) {
                    double term = lm_score_token(lm, lmst[p], k);
                    if (cfg.blank_mode == 1) term += d_log1mexp(asrb[p]);
                    s += cfg.lam * term;
                    atomicAdd(&n_early, 1);
                }
                n_len = ln[p] + 1;
                n_hash = d_update_hash(hs[p], k, cfg.hbase, cfg.hmod);
                n_last = k;
                n_f = cdest[x];
                n_lm = cfg.with_lm ? lm_advance(lm, lmst[p], k) : 0;
                n_tok = k;
                if (col < st.max_cols) {
                    const size_t node = static_cast<size_t>(col) * S + sout;
                    st.st_tok[node] = k;
                    st.st_prev[node] = tn[p];
                    st.st_dur[node] = ND > 0 ? static_cast<signed char>(m.durations[cdi[x]]) : 0;
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
    if (tid == 0 && col < st.max_cols) st.st_frame[static_cast<size_t>(col) * st.B + b] = t;
    __syncthreads();
    // prediction-state pool (2K entries per stream): a blank / dead child keeps
    // its parent's entry (no copy); a token child gets an entry no current slot
    // uses, so the parent's state stays intact for this round's LSTM step
    if (tid == 0) {
        unsigned long long used = 0ull;
        for (int i = 0; i < K; ++i) used |= 1ull << s_pid[i];
        for (int j = 0; j < K; ++j) {
            if (s_tok[j] >= 0) {
                const int e = __ffsll(static_cast<long long>(~used)) - 1;
                used |= 1ull << e;
                s_npid[j] = e;
            } else {
                s_npid[j] = s_pid[s_par[j]];
            }
        }
    }
    __syncthreads();
    if (tid < K) {
        const int j = tid;
        const int sout = b * K + j;
        int upos = -1;
        if (s_tok[j] >= 0 && m.pred_kind == 1) {
            upos = atomicAdd(&st.upd_count[cur], 1);
            st.upd_list[cur * S + upos] = sout;
            st.upd_src[cur * S + upos] = b * st.P + s_pid[s_par[j]];
            st.upd_dst[cur * S + upos] = b * st.P + s_npid[j];
            st.upd_tok[cur * S + upos] = s_tok[j];
        }
        if (st.tc) st.upd_pos[sout] = upos;
        s_upos[j] = upos;
    }
    if (tid < K) {
        sc[tid] = n_score;
        ln[tid] = n_len;
        hs[tid] = n_hash;
        ls[tid] = n_last;
        fr[tid] = n_f;
        tn[tid] = n_tn;
        lmst[tid] = n_lm;
    }
    if (tid == 0) {
        int na = 0;
        for (int i = 0; i < K; ++i) na += act[i];
        n_active = na;
    }
    __syncthreads();

    SEL_MARK(4);
    // 8. stream state machine + counters --------------------------------------------
    __shared__ int s_t, s_done, s_newframe;
    if (tid == 0) {
        unsigned long long* ctr = st.ctr + static_cast<size_t>(b) * 5;
        ctr[1] += 1ull;
        ctr[2] += static_cast<unsigned long long>(n_active);
        if (cfg.late) ctr[4] += static_cast<unsigned long long>(n_active);
        ctr[3] += static_cast<unsigned long long>(n_early);
        int nr = r + 1;
        bool any = false;
        for (int i = 0; i < K; ++i)
            if (sc[i] != -INFINITY && fr[i] == t) any = true;
        int nt = t;
        int newframe = 0;
        if (nr >= cfg.rounds || !any) {
            ctr[0] += 1ull;
            nt = T;
            for (int i = 0; i < K; ++i)
                if (sc[i] != -INFINITY) nt = min(nt, fr[i]);
            if (nt <= t) nt = t + 1;
            nr = 0;
            newframe = 1;
        }
        int done = 0;
        if (nt >= T) {
            done = 1;
            st.steps[b] = col + 1;
            atomicAdd(st.n_done, 1);
        }
        st.col[b] = col + 1;
        st.t[b] = nt;
        st.r[b] = nr;
        st.done[b] = done;
        s_t = nt;
        s_done = done;
        s_newframe = newframe;
    }
    __syncthreads();
    if (tid < K) {
        const int j = tid;
        const size_t s = static_cast<size_t>(b) * K + j;
        st.score[s] = sc[j];
        st.len[s] = ln[j];
        st.hash[s] = hs[j];
        st.last[s] = ls[j];
        st.f[s] = fr[j];
        st.tnode[s] = tn[j];
        st.lm_state[s] = lmst[j];
        st.pid[s] = s_npid[j];
        // aes_pp quirk: per-slot flag, not permuted, reset at frame start only
        st.sdonated[s] = (cfg.quirk && !s_newframe) ? static_cast<unsigned char>(don[j]) : 0;
        int apos = -1;
        if (!s_done && sc[j] != -INFINITY && fr[j] == s_t) {
            apos = atomicAdd(&st.act_count[nxt], 1);
            st.act_list[nxt * S + apos] = static_cast<int>(s);
        }
        if (st.tc) st.act_pos[s] = apos;
        s_apos[j] = apos;
    }
    __syncthreads();
    if (s_done) return;

    SEL_MARK(5);
    // 9. prediction-network state of the new beam, gathered by parent (decoder.cpp
    //    :288-318): blank/dead children copy the parent's state; token children
    //    shift the stateless window (model.cpp:109-121) or -- LSTM -- stage the
    //    parent's h for the gate GEMM.  Every slot active next round also gets
    //    its joint operand z = bf16(tanh(enc_proj[b, t'] + pred)) (tensor-core path).
    const float* ep = st.encp + (static_cast<size_t>(b) * st.Tmax + s_t) * m.J;
    const size_t prow0 = static_cast<size_t>(b) * st.P;  // this stream's pool rows
    if (m.pred_kind == 1) {
        // token children: stage the parent's h (bf16) for the gate GEMM;
        // children active next round that keep their entry: z = tanh(enc + pred)
        const int H4 = m.H >> 2, J4 = m.J >> 2;
        for (int it = tid; it < K * (H4 > J4 ? H4 : J4); it += nthr) {
            const int j = it / (H4 > J4 ? H4 : J4), e = it - j * (H4 > J4 ? H4 : J4);
            if (s_tok[j] >= 0) {
                if (st.tc && e < H4) {
                    const float4 v = reinterpret_cast<const float4*>(st.h + (prow0 + s_pid[s_par[j]]) * m.H)[e];
                    const __nv_bfloat162 a01 = __floats2bfloat162_rn(v.x, v.y);
                    const __nv_bfloat162 a23 = __floats2bfloat162_rn(v.z, v.w);
                    uint2 pk;
                    pk.x = *reinterpret_cast<const uint32_t*>(&a01);
                    pk.y = *reinterpret_cast<const uint32_t*>(&a23);
                    reinterpret_cast<uint2*>(st.hA16 + static_cast<size_t>(s_upos[j]) * st.Hp)[e] = pk;
                }
            } else if (st.tc && s_apos[j] >= 0 && e < J4) {
                const float4 v = reinterpret_cast<const float4*>(st.pred + (prow0 + s_npid[j]) * m.J)[e];
                const float4 ev = reinterpret_cast<const float4*>(ep)[e];
                const __nv_bfloat162 z01 = __floats2bfloat162_rn(tanhf(ev.x + v.x), tanhf(ev.y + v.y));
                const __nv_bfloat162 z23 = __floats2bfloat162_rn(tanhf(ev.z + v.z), tanhf(ev.w + v.w));
                uint2 pk;
                pk.x = *reinterpret_cast<const uint32_t*>(&z01);
                pk.y = *reinterpret_cast<const uint32_t*>(&z23);
                reinterpret_cast<uint2*>(st.z16 + static_cast<size_t>(s_apos[j]) * st.Jp)[e] = pk;
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
        for (int q = 0; q < n; ++q) {
            const int w = q + 1 < n ? wsrc[q + 1] : tok;
            wdst[q] = w;
            if (win_smem) s_win[j * 16 + q] = w;
        }
    }
    __syncthreads();
    const float inv = n > 0 ? 1.0f / n : 0.f;
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
            for (int q = 0; q < n; ++q) {
                const int w = win_smem ? s_win[j * 16 + q] : wl[q];
                acc += inv * m.table[static_cast<size_t>(w < 0 ? m.V : w) * m.J + c];
            }
            v = m.b_pred[c] + acc;
            st.pred[row * m.J + c] = v;
        }
        if (st.tc && apos >= 0) st.z16[static_cast<size_t>(apos) * st.Jp + c] = __float2bfloat16_rn(tanhf(ep[c] + v));
    }
}

// One CTA (256 threads) per stream; the last CTA to finish does the loop
// bookkeeping: list-count resets for the parity double buffers, the round
// counter, and (set_cond) the CUDA-graph WHILE condition "a stream is still
// decoding" -- so the loop needs no control kernel and no host sync.
__global__ void __launch_bounds__(256) select_kernel(DevModel m, DevLm lm, DevCfg cfg, DevState st, int par,
                                                     cudaGraphConditionalHandle hcond, int set_cond) {
    pdl_trigger();
    pdl_wait();
    const long long tk0 = clock64();
    if (!st.done[blockIdx.x]) select_stream(m, lm, cfg, st, par);
    if (g_sel_trace_on && blockIdx.x == 0 && threadIdx.x == 0) {
        g_sel_trace[0] += 1;
        g_sel_trace[7] += clock64() - tk0;
    }
    if (threadIdx.x == 0) {
        if (blockIdx.x == 0) {
            st.act_count[par] = 0;      // read by this round's joint (finished)
            st.upd_count[par ^ 1] = 0;  // read by last round's LSTM GEMMs (finished)
        }
        __threadfence();
        const int k = atomicAdd(st.sel_blocks, 1);
        if (k == static_cast<int>(gridDim.x) - 1) {
            *st.sel_blocks = 0;
            const int rounds = atomicAdd(st.g, 1) + 1;
            const int nd = atomicAdd(st.n_done, 0);
            if (set_cond) cudaGraphSetConditional(hcond, (nd < st.B && rounds < st.max_cols) ? 1u : 0u);
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

void sel_trace(int enable, long long* out) {
    if (out) cudaMemcpyFromSymbol(out, g_sel_trace, sizeof(long long) * 8);
    long long z[8] = {};
    cudaMemcpyToSymbol(g_sel_trace, z, sizeof(z));
    cudaMemcpyToSymbol(g_sel_trace_on, &enable, sizeof(int));
}

void configure_kernels() {
    cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(select_smem_bytes(kMaxBeam, kMaxDur, 2048 / kMaxBeam)));
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
    lc.dynamicSmemBytes = select_smem_bytes(cfg.K, m.ND, st.NT);
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    cudaLaunchKernelEx(&lc, select_kernel, m, lm, cfg, st, par, h, set_cond);
}

void launch_enc_to_bf16(const DevModel& m, const DevState& st, int rows, cudaStream_t s) {
    enc_to_bf16_kernel<<<148 * 8, 256, 0, s>>>(m, st, rows);
}

void launch_finalize(const DevModel& m, const DevLm& lm, const DevCfg& cfg, const DevState& st,
                     cudaStream_t s) {
    finalize_kernel<<<st.B, 32, 0, s>>>(m, lm, cfg, st);
}

}  // namespace tbeam_dev
