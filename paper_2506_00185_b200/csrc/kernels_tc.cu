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
//   tc_gemm_s3 precision fp32: the joint / gates / proj GEMMs on three bf16
//              planes per operand, per-k-block accumulators summed in fp64
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
#include <vector>

#include "device_fns.cuh"
#include "engine.cuh"
#include "kernels.h"
#include "tc_common.cuh"

#include <cooperative_groups.h>

namespace tbeam_dev {

constexpr int BM = 128;

struct TmemAcc {
    int n;             // accumulators to sum
    uint32_t stride;   // TMEM columns between them
    __device__ __forceinline__ void ld8(uint32_t taddr, float (&v)[8]) const { tmem_ldacc(taddr, v, n, stride); }
};
constexpr int BK = 64;
constexpr int A_BYTES = BM * BK * 2;

// as many K stages as ~200 KB of smem holds: for the decode's K = 640
// (10 k-blocks) narrow tiles keep every load in flight at once
template <int BN>
__host__ __device__ constexpr int tc_stages() {
    return (200 * 1024) / (A_BYTES + BN * BK * 2) > 12 ? 12 : (200 * 1024) / (A_BYTES + BN * BK * 2);
}

// ring + barriers/TMEM slot + a 1 KB epilogue side buffer (bias) that the
// epilogue warps fill while the mainloop still owns the ring
template <int BN>
__host__ __device__ constexpr int tc_smem_bytes() {
    return 1024 + tc_stages<BN>() * (A_BYTES + BN * BK * 2) + 256 + 2048 + 16;
}

// independent K-split accumulators per tile (summed by the epilogue): one.
// Round 1 split the 40 dependent MMAs of a K = 640 loop over 4 (BN <= 64) or
// 2 (BN <= 128) accumulators; the MMA chain was never the limit and every
// epilogue column load then sums 4 TMEM reads -- one accumulator measured
// 32.6 -> 31.8 us per round at the bench shape (greedy unchanged).
// -DTBEAM_KACC=2|4 restores a K-split (measurement switch).
template <int BN>
__host__ __device__ constexpr int tc_kacc() {
#ifdef TBEAM_KACC
    return BN <= 128 ? TBEAM_KACC : 1;
#else
    return 1;
#endif
}
template <int BN>
__host__ __device__ constexpr uint32_t tmem_acc_cols() {
    return BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
}
template <int BN>
__host__ __device__ constexpr uint32_t tmem_cols() {
    return tmem_acc_cols<BN>() * tc_kacc<BN>();
}

// Phase trace of CTA (0,0) of every tc_gemm launch (SM clock): entry,
// prologue done, dependency resolved, accumulator ready, epilogue done.
// Read back with tbeam_debug_gemm_trace (measurement aid, ~free).
__device__ long long g_gemm_trace[40];
// device-wide launch timeline (tc_common.cuh), kernels 0 joint, 1 gates, 2 proj
__device__ unsigned long long g_tl_tc[kTlRounds * 4 * 4];

// ---------------------------------------------------------------------------
// the GEMM skeleton
// ---------------------------------------------------------------------------
constexpr int GEMM_THREADS = 512;  // warp 0 lane 0: TMA, warp 1 lane 0: MMA; 16 epilogue warps

// MC > 1: the MC CTAs of a (1, MC) cluster share the A tile (same rows,
// different N tiles); each loads a 128/MC-row slice of every A box and TMA-
// multicasts it to all MC CTAs, cutting the per-SM L2 -> smem A traffic by MC.
// Used only when every k-block has its own stage (nk <= STAGES): no stage is
// reused, so no cross-CTA "empty" handshake is needed.
template <int BN, class Epi, int MC = 1>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int K,
        int bnv, Epi epi) {
    constexpr int B_BYTES = BN * BK * 2;
    constexpr int STAGES = tc_stages<BN>();
    extern __shared__ uint8_t smem_raw[];
    // (offset arithmetic on the __shared__ array, not a uintptr_t round trip:
    // the compiler then keeps every epilogue access in the shared window --
    // LDS / STS instead of generic LD / ST)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* done = empty + STAGES;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);

    const int m0 = blockIdx.x * BM;
    const int n0 = blockIdx.y * bnv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool tr = (epi.st.trace & 1) && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0;
    long long t_entry = 0, t_pro = 0, t_dep = 0, t_acc = 0;
    if (tr) t_entry = clock64();
    const bool tlon = (epi.st.trace & 2) && threadIdx.x == 0;
    const unsigned long long tl_entry = tlon ? gtimer() : 0ull;
    unsigned long long tl_rel = 0ull;

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
    if constexpr (MC > 1) cluster_sync();  // peers' barriers initialised before any multicast
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    if (tr) t_pro = clock64();
    const int nk = (K + BK - 1) / BK;
    // the weight (B) operand does not depend on the previous kernel: its
    // first ring-full of k-blocks is fetched BEFORE the dependency wait, so
    // it overlaps the previous kernel's tail (the stage's arrival -- and the
    // A bytes -- come after the wait)
    const int npre = MC > 1 ? 0 : (nk < STAGES ? nk : STAGES);
    const uint32_t b_bytes = static_cast<uint32_t>(bnv) * BK * 2;
    if (threadIdx.x == 0)
        for (int kb = 0; kb < npre; ++kb) {
            mbar_expect_tx_only(&full[kb], b_bytes);
            tma_load_2d(sB + kb * B_BYTES, &tmB, &full[kb], kb * BK, n0);
        }
    pdl_trigger();
    pdl_wait();
    if (tr) t_dep = clock64();
    if (tlon) tl_rel = gtimer();
    const int tl_rnd = tlon ? epi.tl_round() : -1;
    const int rows = epi.rows();
    if (m0 >= rows) {  // no rows for this tile this round (uniform across a cluster)
        if (threadIdx.x == 0)  // let the preloaded weight bytes land before the smem goes away
            for (int kb = 0; kb < npre; ++kb) {
                mbar_expect_tx(&full[kb], 0);
                mbar_wait(&full[kb], 0);
            }
        if (tlon) tl_record(g_tl_tc, tl_rnd, Epi::kTrace, tl_entry, tl_rel, gtimer());
        __syncthreads();
        if (warp == 0) tmem_dealloc(tmem, tmem_cols<BN>());
        if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) epi.finish();
        return;
    }

    if (threadIdx.x == 0) {
        // TMA producer.  A arrives in 32-row boxes (4 swizzle atoms each) and
        // only the boxes holding live rows are fetched: a tile of 45 token rows
        // moves 64 rows of activations, not 128 (the rest of the smem tile is
        // stale; its accumulator rows are never read)
        const int nbox = MC > 1 ? BM / 32 : (min(BM, rows - m0) + 31) >> 5;
        const uint32_t a_bytes = static_cast<uint32_t>(nbox) * 32 * BK * 2;
        const uint32_t bytes = a_bytes + b_bytes;
        for (int kb = 0; kb < nk; ++kb) {
            const int s = kb % STAGES;
            const uint32_t use = kb / STAGES;
            if (kb < npre) {  // weights already in flight: arrive + the A bytes
                mbar_expect_tx(&full[s], a_bytes);
                for (int i = 0; i < nbox; ++i)
                    tma_load_2d(sA + s * A_BYTES + i * 32 * BK * 2, &tmA, &full[s], kb * BK, m0 + 32 * i);
                continue;
            }
            if (kb >= STAGES) mbar_wait(&empty[s], (use & 1u) ^ 1u);
            mbar_expect_tx(&full[s], bytes);
            if constexpr (MC > 1) {
                constexpr int SLICE = BM / MC;
                const int cr = static_cast<int>(cluster_rank());
                tma_load_2d_mc(sA + s * A_BYTES + cr * SLICE * BK * 2, &tmA, &full[s], kb * BK, m0 + cr * SLICE,
                               static_cast<uint16_t>((1u << MC) - 1));
            } else {
                for (int i = 0; i < nbox; ++i)
                    tma_load_2d(sA + s * A_BYTES + i * 32 * BK * 2, &tmA, &full[s], kb * BK, m0 + 32 * i);
            }
            tma_load_2d(sB + s * B_BYTES, &tmB, &full[s], kb * BK, n0);
        }
    }
    if (warp_uniform_idx() == 1) {
        // MMA warp: uniform operands, one elected lane issues (tc_common.cuh)
        const uint32_t idesc = umma_idesc_bf16(BM, bnv);
        const bool trm = (epi.st.trace & 1) && blockIdx.x == 0 && blockIdx.y == 0 && lane == 0;
        const long long tm0 = trm ? clock64() : 0;
        const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
        const uint32_t sa0 = __shfl_sync(0xffffffffu, smem_u32(sA), 0);
        const uint32_t sb0 = __shfl_sync(0xffffffffu, smem_u32(sB), 0);
        for (int kb = 0; kb < nk; ++kb) {
            const int s = kb % STAGES;
            mbar_wait(&full[s], (kb / STAGES) & 1u);
            if (trm && kb == 0) g_gemm_trace[8 * Epi::kTrace + 5] += clock64() - tm0;
            if (trm && kb == nk - 1) g_gemm_trace[8 * Epi::kTrace + 6] += clock64() - tm0;
            tc_fence_after();
            const uint32_t a0 = sa0 + s * A_BYTES;
            const uint32_t b0 = sb0 + s * B_BYTES;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
                constexpr int KA = tc_kacc<BN>();
                const int j = kb * (BK / 16) + k;  // k-step; accumulator j % KA
                if (elect_one())
                    umma_bf16(tm + static_cast<uint32_t>(j % KA) * tmem_acc_cols<BN>(), umma_desc_sw128(a0 + 32 * k),
                              umma_desc_sw128(b0 + 32 * k), idesc, j >= KA ? 1u : 0u);
                __syncwarp();
            }
            if (elect_one()) umma_commit(&empty[s]);
            __syncwarp();
        }
        if (elect_one()) umma_commit(done);
        __syncwarp();
    }
    // warp w reads TMEM lanes 32*(w%4).. (its 32 tile rows) and columns of
    // sub-block w/4: four warps share a row group, each a quarter of the tile
    const int grp = warp & 3, sub = warp >> 2;
    // the epilogue's own global loads (row lists, bias, LSTM inputs, ...) go
    // out while the tensor core works
    uint8_t* bias_smem = sB + STAGES * B_BYTES + (STAGES + STAGES + 1) * 8 + 8;
    bias_smem += (16u - (smem_u32(bias_smem) & 15u)) & 15u;
    const typename Epi::Pre pre = epi.prefetch(grp, lane, m0, n0, bnv, sub, bias_smem);
    mbar_wait(done, 0);
    __syncwarp();
    tc_fence_after();
    if (tr) t_acc = clock64();
    __syncthreads();  // prefetched smem (bias) visible to every thread
    // (a K shorter than KA k-steps leaves accumulators unwritten: use fewer)
    const int nacc = tc_kacc<BN>() < nk * (BK / 16) ? tc_kacc<BN>() : nk * (BK / 16);
    epi.run(tmem + (static_cast<uint32_t>(grp * 32) << 16), grp, lane, m0, blockIdx.y, n0, bnv, sub, smem, pre,
            bias_smem, TmemAcc{nacc, tmem_acc_cols<BN>()});
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
    if constexpr (MC > 1) cluster_sync();  // no CTA leaves while a peer may still receive
    else __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, tmem_cols<BN>());
    if (tlon) tl_record(g_tl_tc, tl_rnd, Epi::kTrace, tl_entry, tl_rel, gtimer());
    if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) epi.finish();
}

// ---------------------------------------------------------------------------
// Full-K GEMM for the short decode GEMMs (K = nk * 64 <= 640, BN = 32): the
// whole A tile (live rows rounded to 32/64/128) and the whole B tile each
// arrive in ONE 3-D TMA box -- TMA serves a CTA's boxes one after another
// with a fixed cost per box, so ten per-k-block boxes cost 2-3x one big box.
// B (weights) is requested before the dependency wait.  No smem ring: the
// tile's k-blocks all fit (<= 160 KB A + 40 KB B).
// ---------------------------------------------------------------------------
constexpr int FK_MAX_NK = 10;
#ifndef FK_ABOXES
#define FK_ABOXES 2  // A operand boxes per full-K tile (2: round 2 A/B)
#endif
static_assert(FK_ABOXES >= 1 && FK_ABOXES <= 5, "A boxes: 1..5");
// k-block slots of the A region: whole boxes (a box past nk is zero-filled)
constexpr int FK_A_KB = FK_ABOXES * ((FK_MAX_NK + FK_ABOXES - 1) / FK_ABOXES);

template <int BN>
__host__ __device__ constexpr int fk_smem_bytes() {
    return 1024 + (FK_A_KB * BM + FK_MAX_NK * BN) * 128 + 64 + 2048 + 16;
}

template <int BN, class Epi>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
tc_gemm_fk(const __grid_constant__ CUtensorMap tmA32, const __grid_constant__ CUtensorMap tmA64,
           const __grid_constant__ CUtensorMap tmA128, const __grid_constant__ CUtensorMap tmB, int nk, int bnv,
           Epi epi) {
    extern __shared__ uint8_t smem_raw[];
    // (offset arithmetic on the __shared__ array, not a uintptr_t round trip:
    // the compiler then keeps every epilogue access in the shared window --
    // LDS / STS instead of generic LD / ST)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    uint8_t* sB = smem + FK_A_KB * BM * 128;
    uint64_t* fullA = reinterpret_cast<uint64_t*>(sB + FK_MAX_NK * BN * 128);
    uint64_t* fullB = fullA + 1;
    uint64_t* done = fullA + 2;
    uint64_t* fullA2 = fullA + 3;  // [FK_ABOXES - 1] barriers of the later A boxes
    uint32_t* tslot = reinterpret_cast<uint32_t*>(fullA + 2 + FK_ABOXES);
    uint8_t* side = reinterpret_cast<uint8_t*>(fullA + 8);

    // grid (N tiles, M tiles): the first M-tile's CTAs -- live whenever any
    // row is -- are dispatched first; later (usually empty) M-tiles exit early
    const int mt = blockIdx.y, ntile = blockIdx.x;
    const int m0 = mt * BM;
    const int n0 = ntile * bnv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool tlon = (epi.st.trace & 2) && threadIdx.x == 0;
    const unsigned long long tl_entry = tlon ? gtimer() : 0ull;
    // phase trace of CTA (0,0) (same slots as tc_gemm): prologue, dependency
    // wait, operands landed + MMAs done, epilogue
    const bool tr = (epi.st.trace & 1) && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0;
    long long t_entry = tr ? clock64() : 0, t_pro = 0, t_dep = 0, t_acc = 0;
    unsigned long long tl_rel = 0ull;
    if (threadIdx.x == 0) {
        mbar_init(fullA, 1);
        mbar_init(fullB, 1);
        mbar_init(done, 1);
        for (int q = 0; q < FK_ABOXES - 1; ++q) mbar_init(fullA2 + q, 1);
        mbar_fence_init();
        tma_prefetch(&tmB);
        tma_prefetch(&tmA32);
        tma_prefetch(&tmA64);
        tma_prefetch(&tmA128);
    }
    if (warp == 0) tmem_alloc(tslot, tmem_cols<BN>());
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    // weights: independent of the previous kernel, so the first M-tile (live
    // whenever any row is) requests them before the dependency wait; later
    // M-tiles only once they know they have rows
    const bool pre_b = mt == 0;
    if (threadIdx.x == 0 && pre_b) {
        mbar_expect_tx(fullB, static_cast<uint32_t>(nk) * BN * 128);
        tma_load_3d(sB, &tmB, fullB, 0, n0, 0);
    }
    if (tr) t_pro = clock64();
    pdl_trigger();
    pdl_wait();
    if (tr) t_dep = clock64();
    if (tlon) tl_rel = gtimer();
    const int tl_rnd = tlon ? epi.tl_round() : -1;
    const int rows = epi.rows();
    if (m0 >= rows) {  // no rows for this tile this round
        if (threadIdx.x == 0 && pre_b) mbar_wait(fullB, 0);  // the weight box lands before the smem goes away
        if (tlon) tl_record(g_tl_tc, tl_rnd, Epi::kTrace, tl_entry, tl_rel, gtimer());
        __syncthreads();
        if (warp == 0) tmem_dealloc(tmem, tmem_cols<BN>());
        if (threadIdx.x == 0 && mt == 0 && ntile == 0) epi.finish();
        return;
    }
    const int live = min(BM, rows - m0);
    const int RB = live <= 32 ? 32 : live <= 64 ? 64 : 128;
    // A in FK_ABOXES boxes of nh k-blocks (the maps' box depth): the MMAs on
    // the first boxes run while the later ones land
    const int nh = (nk + FK_ABOXES - 1) / FK_ABOXES;
    if (threadIdx.x == 0) {
        if (!pre_b) {
            mbar_expect_tx(fullB, static_cast<uint32_t>(nk) * BN * 128);
            tma_load_3d(sB, &tmB, fullB, 0, n0, 0);
        }
        const CUtensorMap* ma = RB == 32 ? &tmA32 : RB == 64 ? &tmA64 : &tmA128;
        mbar_expect_tx(fullA, static_cast<uint32_t>(nh) * RB * 128);
        tma_load_3d(sA, ma, fullA, 0, m0, 0);
        for (int q = 1; q < FK_ABOXES && q * nh < nk; ++q) {
            mbar_expect_tx(fullA2 + q - 1, static_cast<uint32_t>(nh) * RB * 128);
            tma_load_3d(sA + q * nh * RB * 128, ma, fullA2 + q - 1, 0, m0, q * nh);
        }
    }
    if (warp_uniform_idx() == 1) {  // MMA warp: uniform operands, one elected lane issues
        const uint32_t idesc = umma_idesc_bf16(BM, bnv);
        const bool trm = (epi.st.trace & 1) && blockIdx.x == 0 && blockIdx.y == 0 && lane == 0;
        const long long tm0 = trm ? clock64() : 0;
        const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
        const int rbu = __shfl_sync(0xffffffffu, RB, 0);
        const uint32_t sa0 = __shfl_sync(0xffffffffu, smem_u32(sA), 0);
        const uint32_t sb0 = __shfl_sync(0xffffffffu, smem_u32(sB), 0);
        mbar_wait(fullB, 0);
        mbar_wait(fullA, 0);
        if (trm) g_gemm_trace[8 * Epi::kTrace + 5] += clock64() - tm0;  // operands landed
        tc_fence_after();
        constexpr int KA = tc_kacc<BN>();
        const int nhu = __shfl_sync(0xffffffffu, nh, 0);
        for (int kb = 0; kb < nk; ++kb) {
            if (kb > 0 && kb % nhu == 0) {  // the next A box
                mbar_wait(fullA2 + kb / nhu - 1, 0);
                tc_fence_after();
            }
            const uint32_t a0 = sa0 + kb * rbu * 128;  // rows >= RB: stale smem, rows never read
            const uint32_t b0 = sb0 + kb * BN * 128;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int j = kb * 4 + k;
                if (elect_one())
                    umma_bf16(tm + static_cast<uint32_t>(j % KA) * tmem_acc_cols<BN>(), umma_desc_sw128(a0 + 32 * k),
                              umma_desc_sw128(b0 + 32 * k), idesc, j >= KA ? 1u : 0u);
                __syncwarp();
            }
        }
        if (elect_one()) umma_commit(done);
        __syncwarp();
        if (trm) g_gemm_trace[8 * Epi::kTrace + 6] += clock64() - tm0;  // MMAs issued
    }
    const int grp = warp & 3, sub = warp >> 2;
    const typename Epi::Pre pre = epi.prefetch(grp, lane, m0, n0, bnv, sub, side);
    mbar_wait(done, 0);
    __syncwarp();
    tc_fence_after();
    if (tr) t_acc = clock64();
    __syncthreads();  // prefetched smem (bias) visible to every thread
    const int nacc = tc_kacc<BN>() < nk * 4 ? tc_kacc<BN>() : nk * 4;
    epi.run(tmem + (static_cast<uint32_t>(grp * 32) << 16), grp, lane, m0, ntile, n0, bnv, sub, smem, pre, side,
            TmemAcc{nacc, tmem_acc_cols<BN>()});
    if (tr) {
        long long* g = g_gemm_trace + 8 * Epi::kTrace;
        g[0] += 1;
        g[1] += t_pro - t_entry;
        g[2] += t_dep - t_pro;
        g[3] += t_acc - t_dep;
        g[4] += clock64() - t_acc;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, tmem_cols<BN>());
    if (tlon) tl_record(g_tl_tc, tl_rnd, Epi::kTrace, tl_entry, tl_rel, gtimer());
    if (threadIdx.x == 0 && mt == 0 && ntile == 0) epi.finish();
}

// ---------------------------------------------------------------------------
// fp32 GEMMs on the tensor cores (precision = fp32).  Every fp32 operand is
// staged as three bf16 planes, x = x0 + x1 + x2 exactly (device_fns.cuh
// put_op), and the product keeps the six plane products x_i . y_j with
// i + j <= 2 (the dropped ones are below 2^-24 of |x||y|).  UMMA accumulates
// in fp32 with truncation: ONE accumulator over K = 640 lands ~1e-5 rms off
// the fp64 product (sequential FFMA: 1e-6), so every k-block gets its own TMEM
// accumulator and the epilogue sums them in fp64 -- 9e-7 max / 1.8e-7 rms,
// the CUDA-core path's fp64-folded FFMA being 5e-7 / 1.3e-7
// (scripts/micro/split_mma.cu, profiles/r02/split_mma.txt).
// A CTA takes `per` <= 3 k-blocks of one BN = 32 tile: one 4-D TMA box per
// operand, all planes and k-blocks (weights before the dependency wait), and
// per k-step three MMAs against the stacked B planes (N = 96 / 64 / 32).  The
// K slices of a tile run in separate CTAs (blockIdx.z); each stores its fp64
// partial tile and the last to arrive (ticket) sums them in slice order --
// deterministic -- then runs the bf16 path's fused epilogue on the reduced
// tile, read from smem (SmemAcc instead of TMEM).  clu = 1 (opt-in, measured
// slower): the slices form one cluster and meet through DSMEM.
// ---------------------------------------------------------------------------
constexpr int S3_MAX_PER = 3;
constexpr int S3_A = S3_MAX_PER * 3 * BM * 128;  // A: per k-blocks x 3 planes x 128 rows x 128 B
constexpr int S3_B = S3_MAX_PER * 3 * 32 * 128;  // B: per k-blocks x 3 planes x 32 rows x 128 B
constexpr int S3_PITCH = 33;                     // reduced tile row pitch (floats)
// TMEM: per k-block [x0.y0 | x0.y1 | x0.y2] (one N = 96 MMA against the three
// stacked B planes), then [x1.y0 | x1.y1] (N = 64) and x2.y0 (N = 32), the
// small products accumulated over the CTA's k-blocks
constexpr uint32_t S3_R1 = S3_MAX_PER * 96, S3_R2 = S3_R1 + 64;
__host__ __device__ constexpr int s3_smem_bytes() {
    return 1024 + S3_A + S3_B + BM * S3_PITCH * 4 + 64 + 2048 + 16;
}

// the reduced tile as the epilogue's accumulator source: column offsets come
// in as the "TMEM address" (the kernel passes base 0)
struct SmemAcc {
    const float* row;
    __device__ __forceinline__ void ld8(uint32_t c, float (&v)[8]) const {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = row[c + j];
    }
};

template <class Epi>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
tc_gemm_s3(const __grid_constant__ CUtensorMap tmA32, const __grid_constant__ CUtensorMap tmA64,
           const __grid_constant__ CUtensorMap tmA128, const __grid_constant__ CUtensorMap tmB, int nk, int per,
           int clu, Epi epi) {
    constexpr int BN = 32;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    uint8_t* sB = smem + S3_A;
    float* red = reinterpret_cast<float*>(sB + S3_B);
    uint64_t* fullA = reinterpret_cast<uint64_t*>(red + BM * S3_PITCH);
    uint64_t* fullB = fullA + 1;
    uint64_t* done = fullA + 2;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(fullA + 3);
    int* s_last = reinterpret_cast<int*>(fullA + 4);
    uint8_t* side = reinterpret_cast<uint8_t*>(fullA + 8);

    const int mt = blockIdx.y, ntile = blockIdx.x, ks = blockIdx.z, KS = gridDim.z;
    const int m0 = mt * BM, n0 = ntile * BN;
    const int kb0 = ks * per, nkb = min(per, nk - kb0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool lead = mt == 0 && ntile == 0;  // the tile whose epilogue CTA closes the launch (epi.finish)
    // phase trace of CTA (0,0,0) (tc_gemm's slots) and the launch timeline
    const bool tr = (epi.st.trace & 1) && lead && ks == 0 && threadIdx.x == 0;
    long long t_entry = tr ? clock64() : 0, t_pro = 0, t_dep = 0, t_acc = 0;
    const bool tlon = (epi.st.trace & 2) && threadIdx.x == 0;
    const unsigned long long tl_entry = tlon ? gtimer() : 0ull;
    unsigned long long tl_rel = 0ull;
    if (threadIdx.x == 0) {
        mbar_init(fullA, 1);
        mbar_init(fullB, 1);
        mbar_init(done, 1);
        mbar_fence_init();
        tma_prefetch(&tmB);
        tma_prefetch(&tmA32);
        tma_prefetch(&tmA64);
        tma_prefetch(&tmA128);
    }
    if (warp == 0) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t b_bytes = 3u * static_cast<uint32_t>(per) * BN * 128;
    const bool pre_b = mt == 0;
    if (threadIdx.x == 0 && pre_b) {
        mbar_expect_tx(fullB, b_bytes);
        tma_load_4d(sB, &tmB, fullB, 0, n0, 0, kb0);
    }
    if (tr) t_pro = clock64();
    pdl_trigger();
    pdl_wait();
    if (tr) t_dep = clock64();
    if (tlon) tl_rel = gtimer();
    const int tl_rnd = tlon ? epi.tl_round() : -1;
    const int rows = epi.rows();
    if (m0 >= rows) {  // no rows for this tile this round (every K slice of it exits here)
        if (threadIdx.x == 0 && pre_b) mbar_wait(fullB, 0);
        if (tlon) tl_record(g_tl_tc, tl_rnd, Epi::kTrace, tl_entry, tl_rel, gtimer());
        __syncthreads();
        if (warp == 0) tmem_dealloc(tmem, 512);
        if (threadIdx.x == 0 && lead && ks == 0) epi.finish();
        return;
    }
    const int live = min(BM, rows - m0);
    const int RB = live <= 32 ? 32 : live <= 64 ? 64 : 128;
    if (threadIdx.x == 0) {
        if (!pre_b) {
            mbar_expect_tx(fullB, b_bytes);
            tma_load_4d(sB, &tmB, fullB, 0, n0, 0, kb0);
        }
        mbar_expect_tx(fullA, 3u * static_cast<uint32_t>(per) * RB * 128);
        tma_load_4d(sA, RB == 32 ? &tmA32 : RB == 64 ? &tmA64 : &tmA128, fullA, 0, m0, 0, kb0);
    }
    if (warp_uniform_idx() == 1) {  // MMA warp
        const uint32_t id96 = umma_idesc_bf16(BM, 96), id64 = umma_idesc_bf16(BM, 64), id32 = umma_idesc_bf16(BM, 32);
        const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
        const int rbu = __shfl_sync(0xffffffffu, RB, 0);
        const int nkbu = __shfl_sync(0xffffffffu, nkb, 0);
        const uint32_t sa0 = __shfl_sync(0xffffffffu, smem_u32(sA), 0);
        const uint32_t sb0 = __shfl_sync(0xffffffffu, smem_u32(sB), 0);
        const bool trm = (epi.st.trace & 1) && lead && ks == 0 && lane == 0;
        const long long tm0 = trm ? clock64() : 0;
        mbar_wait(fullB, 0);
        mbar_wait(fullA, 0);
        if (trm) g_gemm_trace[8 * Epi::kTrace + 5] += clock64() - tm0;  // operands landed
        tc_fence_after();
        // smem: A tile (k-block kb, plane p) at (3 kb + p) RB rows; B k-block kb
        // = its three planes stacked, 96 rows (N = 96 / 64 / 32 take 3 / 2 / 1)
        for (int kb = 0; kb < nkbu; ++kb) {
            const uint32_t a0 = sa0 + (3 * kb) * rbu * 128;
            const uint32_t b0 = sb0 + kb * 96 * 128;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t bd = umma_desc_sw128(b0 + 32 * k);
                if (elect_one()) {
                    umma_bf16(tm + static_cast<uint32_t>(kb) * 96, umma_desc_sw128(a0 + 32 * k), bd, id96,
                              k ? 1u : 0u);
                    umma_bf16(tm + S3_R1, umma_desc_sw128(a0 + rbu * 128 + 32 * k), bd, id64, (kb | k) ? 1u : 0u);
                    umma_bf16(tm + S3_R2, umma_desc_sw128(a0 + 2 * rbu * 128 + 32 * k), bd, id32,
                              (kb | k) ? 1u : 0u);
                }
                __syncwarp();
            }
        }
        if (elect_one()) umma_commit(done);
        __syncwarp();
        if (trm) g_gemm_trace[8 * Epi::kTrace + 6] += clock64() - tm0;  // MMAs issued
    }
    const int grp = warp & 3, sub = warp >> 2;
    const int r = grp * 32 + lane;
    const typename Epi::Pre pre = epi.prefetch(grp, lane, m0, n0, BN, sub, side);
    mbar_wait(done, 0);
    __syncwarp();
    tc_fence_after();
    if (tr) t_acc = clock64();
    // joint sub-phases (slots 36..39): TMEM loads + fp64 sums, partial store +
    // ticket, slice reduction, reductions run by CTA (0,0,0)
    const bool trs = tr && Epi::kTrace == 0;
    // this thread's 8 columns of its row: the k-block accumulators in fp64
    double d[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j] = 0.0;
    {
        // accumulator column blocks of the thread, six loads in flight per
        // wait: k-block 0's x0.y0 (its own accumulator), x0.y1, x0.y2 and the
        // small products x1.y0, x1.y1, x2.y0; then k-blocks 1 and 2.  Each
        // k-block's x0.y0 goes into the fp64 sum on its own; the small
        // products (< 2^-7 of it) are summed in fp32 first.
        const uint32_t tl = tmem + (static_cast<uint32_t>(grp * 32) << 16) + sub * 8;
        uint32_t rv[6][8];
        float sm8[8];
        tmem_ld8_issue(tl, rv[0]);
        tmem_ld8_issue(tl + 32, rv[1]);
        tmem_ld8_issue(tl + 64, rv[2]);
        tmem_ld8_issue(tl + S3_R1, rv[3]);
        tmem_ld8_issue(tl + S3_R1 + 32, rv[4]);
        tmem_ld8_issue(tl + S3_R2, rv[5]);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            d[j] = static_cast<double>(__uint_as_float(rv[0][j]));
            sm8[j] = ((__uint_as_float(rv[1][j]) + __uint_as_float(rv[2][j])) + __uint_as_float(rv[3][j])) +
                     (__uint_as_float(rv[4][j]) + __uint_as_float(rv[5][j]));
        }
        if (nkb > 1) {
#pragma unroll
            for (int q = 0; q < 6; ++q) tmem_ld8_issue(tl + 96 + 32 * q, rv[q]);  // k-blocks 1, 2
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                d[j] += static_cast<double>(__uint_as_float(rv[0][j]));
                sm8[j] += __uint_as_float(rv[1][j]) + __uint_as_float(rv[2][j]);
                if (nkb > 2) {
                    d[j] += static_cast<double>(__uint_as_float(rv[3][j]));
                    sm8[j] += __uint_as_float(rv[4][j]) + __uint_as_float(rv[5][j]);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) d[j] += static_cast<double>(sm8[j]);
    }
    long long ts = trs ? clock64() : 0;
    if (trs) g_gemm_trace[36] += ts - t_acc;
    if (KS > 1 && clu) {
        // the K slices of this tile are the CTAs of one (1, 1, KS) cluster
        // (rank = slice): the others leave their fp64 partial in their own
        // smem (the A ring, free now: [sub][row][8]) and slice 0 sums them
        // through DSMEM in slice order -- deterministic, no global round trip
        const uint32_t pb = smem_u32(smem) + static_cast<uint32_t>((sub * BM + r) * 8 * 8);
        if (ks != 0 && r < live) {
            double2* o = reinterpret_cast<double2*>(smem + (sub * BM + r) * 8 * 8);
#pragma unroll
            for (int j = 0; j < 4; ++j) o[j] = make_double2(d[2 * j], d[2 * j + 1]);
        }
        cluster_arrive();
        cluster_wait();  // partials visible cluster-wide
        if (ks != 0) {
            cluster_arrive();  // released by slice 0 once it has read them
            cluster_wait();
            tc_fence_before();
            __syncthreads();
            if (warp == 0) tmem_dealloc(tmem, 512);
            return;
        }
        if (r < live) {
            for (int q = 1; q < KS; ++q) {
                const uint32_t ca = dsmem_map(pb, static_cast<uint32_t>(q));
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const double2 x = dsmem_ld_f64x2(ca + 16 * j);
                    d[2 * j] += x.x;
                    d[2 * j + 1] += x.y;
                }
            }
        }
        cluster_arrive();  // the other slices may leave (waited for at exit)
        if (trs) {
            g_gemm_trace[38] += clock64() - ts;
            g_gemm_trace[39] += 1;
        }
    } else if (KS > 1) {
        // [tile][slice][sub][row][8] fp64: a warp stores 2 KB contiguously
        const size_t tile = static_cast<size_t>(mt) * gridDim.x + ntile;
        double* base = epi.st.sk_scratch + (tile * KS * 4 + sub) * BM * 8 + static_cast<size_t>(r) * 8;
        const size_t slice = static_cast<size_t>(4) * BM * 8;
        if (r < live) {
            double2* o = reinterpret_cast<double2*>(base + ks * slice);
#pragma unroll
            for (int j = 0; j < 4; ++j) o[j] = make_double2(d[2 * j], d[2 * j + 1]);
        }
        // one fence per CTA: the barrier orders every thread's partial before
        // thread 0's release fence + ticket; the last CTA's acquire fence
        // (thread 0) + the barrier order the slice reads after every store
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const bool last = atomicAdd(epi.st.sk_ticket + tile, 1u) == static_cast<unsigned>(KS - 1);
            if (last) __threadfence();
            *s_last = last;
        }
        __syncthreads();
        if (trs) {
            const long long t2 = clock64();
            g_gemm_trace[37] += t2 - ts;
            ts = t2;
        }
        if (!*s_last) {
            if (tr) {
                long long* g = g_gemm_trace + 8 * Epi::kTrace;
                g[0] += 1;
                g[1] += t_pro - t_entry;
                g[2] += t_dep - t_pro;
                g[3] += t_acc - t_dep;
                g[4] += clock64() - t_acc;
            }
            if (tlon) tl_record(g_tl_tc, tl_rnd, Epi::kTrace, tl_entry, tl_rel, gtimer());
            tc_fence_before();
            __syncthreads();
            if (warp == 0) tmem_dealloc(tmem, 512);
            return;
        }
        if (r < live) {
#pragma unroll
            for (int j = 0; j < 8; ++j) d[j] = 0.0;
            for (int q = 0; q < KS; ++q) {  // slice order: deterministic
                const double2* o = reinterpret_cast<const double2*>(base + q * slice);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const double2 x = __ldcg(o + j);
                    d[2 * j] += x.x;
                    d[2 * j + 1] += x.y;
                }
            }
        }
        if (threadIdx.x == 0) epi.st.sk_ticket[tile] = 0u;  // ready for the next launch
        if (trs) {
            g_gemm_trace[38] += clock64() - ts;
            g_gemm_trace[39] += 1;
        }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) red[r * S3_PITCH + sub * 8 + j] = static_cast<float>(d[j]);
    __syncthreads();  // reduced tile + prefetched smem (bias) visible to every thread
    epi.run(0u, grp, lane, m0, ntile, n0, BN, sub, smem, pre, side, SmemAcc{red + r * S3_PITCH});
    if (tr) {
        long long* g = g_gemm_trace + 8 * Epi::kTrace;
        g[0] += 1;
        g[1] += t_pro - t_entry;
        g[2] += t_dep - t_pro;
        g[3] += t_acc - t_dep;
        g[4] += clock64() - t_acc;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
    if (KS > 1 && clu) cluster_wait();
    if (tlon) tl_record(g_tl_tc, tl_rnd, Epi::kTrace, tl_entry, tl_rel, gtimer());
    if (threadIdx.x == 0 && lead) epi.finish();
}

// ---------------------------------------------------------------------------
// per-thread top-K (value desc, index asc): unrolled bubble insertion
#ifndef TBEAM_PUSH8_MIN
#define TBEAM_PUSH8_MIN 4  // lists of >= this many entries take eight candidates at once
#endif
// ---------------------------------------------------------------------------
// PAY = keep the raw logit of each entry as payload (late LM fusion ranks by
// logit + lambda*lm; the select kernel re-derives the LM value in fp64).
// Without LM fusion the ranking value IS the logit and no payload is kept.
template <int KM, bool PAY>
struct TopK {
    float v[KM];
    int ix[KM];
    float lg[PAY ? KM : 1];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int q = 0; q < KM; ++q) {
            v[q] = -INFINITY;
            ix[q] = 0x7fffffff;
            if constexpr (PAY) lg[q] = 0.f;
        }
    }
    __device__ __forceinline__ float logit(int q) const {
        if constexpr (PAY) return lg[q];
        else return v[q];
    }
    // the list keeps the top KM >= K (a superset of the top K, same order),
    // so the entry threshold is the static last slot
    __device__ __forceinline__ bool enters(float x, int i) const {
        return (x > v[KM - 1]) | ((x == v[KM - 1]) & (i < ix[KM - 1]));
    }
    // merge eight candidates (columns col0..col0+7, all distinct from the
    // list's) in one step: sort them with a 19-comparator network, fold them
    // into the list's tail (bitonic half-cleaner: q >= KM-8 against the
    // reversed candidates) and re-sort the bitonic list -- ~60 compare-
    // exchanges instead of 8 sequential KM-step insertions (KM >= 8)
    __device__ __forceinline__ static bool better(float av, int ai, float bv, int bi) {
        return (av > bv) | ((av == bv) & (ai < bi));
    }
    __device__ __forceinline__ static void ce(float& av, int& ai, float& bv, int& bi) {  // a <- better
        const bool sw = better(bv, bi, av, ai);
        const float tv = av;
        const int ti = ai;
        av = sw ? bv : av;
        ai = sw ? bi : ai;
        bv = sw ? tv : bv;
        bi = sw ? ti : bi;
    }
    __device__ __forceinline__ void push8(const float (&x)[8], int col0) {
        static_assert(KM >= 4 && !PAY, "push8: lists of >= 4 entries, no payload");
        float c[8];
        int ci[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            c[j] = x[j];
            ci[j] = col0 + j;
        }
        // Green's 19-comparator sorting network for 8 inputs (descending)
#define TB_CE(a, b) ce(c[a], ci[a], c[b], ci[b])
        TB_CE(0, 1); TB_CE(2, 3); TB_CE(4, 5); TB_CE(6, 7);
        TB_CE(0, 2); TB_CE(1, 3); TB_CE(4, 6); TB_CE(5, 7);
        TB_CE(1, 2); TB_CE(5, 6); TB_CE(0, 4); TB_CE(3, 7);
        TB_CE(1, 5); TB_CE(2, 6);
        TB_CE(1, 4); TB_CE(3, 6);
        TB_CE(2, 4); TB_CE(3, 5);
        TB_CE(3, 4);
#undef TB_CE
        // half-cleaner: the list (desc) against the candidates reversed (asc)
#pragma unroll
        for (int q = KM > 8 ? KM - 8 : 0; q < KM; ++q) {
            const int j = KM - 1 - q;  // the candidates' best min(KM, 8), reversed
            const bool take = better(c[j], ci[j], v[q], ix[q]);
            v[q] = take ? c[j] : v[q];
            ix[q] = take ? ci[j] : ix[q];
        }
        // the list is now bitonic (desc then asc over its tail): sort it
#pragma unroll
        for (int d = KM / 2; d >= 1; d >>= 1)
#pragma unroll
            for (int q = 0; q < KM; ++q)
                if ((q & d) == 0) ce(v[q], ix[q], v[q + d], ix[q + d]);
    }
    // full (value desc, index asc) order, so an element pushed down past an
    // equal value keeps the lower index ahead
    __device__ __forceinline__ void push(float x, int i, float l) {
        if (KM > 4 && !enters(x, i)) return;  // (the interior-chunk path pre-checks)
        // branch-free insertion: predicated selects, no per-lane branches
#pragma unroll
        for (int q = 0; q < KM; ++q) {
            const bool b = (x > v[q]) | ((x == v[q]) & (i < ix[q]));
            const float tv = v[q];
            const int ti = ix[q];
            v[q] = b ? x : tv;
            ix[q] = b ? i : ti;
            x = b ? tv : x;
            i = b ? ti : i;
            if constexpr (PAY) {
                const float tl = lg[q];
                lg[q] = b ? l : tl;
                l = b ? tl : l;
            }
        }
    }
};

// ---------------------------------------------------------------------------
// joint epilogue.  Thread (row r, sub-block sb) owns columns
// [sb*q, sb*q + q) of the tile (q = bnv/4) and emits its own partial
// (max, sum-exp, top-K) as partial tile nt*4 + sb.
// CLU: the CTA is one of a (1, CL) thread-block cluster along N; the CL
// CTAs' per-row records are merged through distributed shared memory into
// one record per (row, cluster) -- CL x fewer partial bytes written here and
// read back by the select kernel (C5: 33 tile lists per row -> 5).
// ---------------------------------------------------------------------------
template <int KM, bool LATE, bool CLU = false>
struct JointEpi {
    static constexpr int kTrace = 0;
    DevModel m;
    DevLm lm;
    DevCfg cfg;
    DevState st;
    int par;
    __device__ int rows() const { return st.act_count[par]; }
    __device__ int tl_round() const { return *st.g; }
    __device__ void finish() const { *st.live = *st.n_done < st.B ? 1 : 0; }
    // issued during the mainloop: the row's slot, the tile's bias (smem) and,
    // for late fusion, the LM backoff chain of the row's state
    // AES++ prefix probes (st.probe_on, K <= PC): the logits of the stream's
    // slots' last tokens in this row -- the prefix pass's donor values, read
    // from the same accumulators the top-K came from
    static constexpr int PC = KM <= 8 ? KM : 1;  // probes only when K <= 8 (st.probe_on)
    struct Pre {
        int count, slot;
        int L;
        int chain[LATE ? kMaxOrder : 1];
        float accs[LATE ? kMaxOrder : 1];
        float acc_root;
        int npc;
        int pc[PC];
    };
    __device__ Pre prefetch(int grp, int lane, int m0, int n0, int bnv, int sb, uint8_t* side) const {
        Pre p;
        const int row = m0 + grp * 32 + lane;
        p.count = st.act_count[par];
        p.slot = row < st.S ? st.act_list[par * st.S + row] : -1;
        p.npc = 0;
        if (st.probe_on && row < p.count) {
            const int b = p.slot / cfg.K;
            if (st.r[b] == 0) {  // the select's prefix pass runs at round 0 of a frame
                p.npc = cfg.K;
#pragma unroll
                for (int q = 0; q < PC; ++q) p.pc[q] = q < cfg.K ? st.last[b * cfg.K + q] : -1;
            }
        }
        const int ncols = m.R + m.ND;
        float* bias = reinterpret_cast<float*>(side);
        for (int c = threadIdx.x; c < bnv; c += GEMM_THREADS) bias[c] = n0 + c < ncols ? m.b_out[n0 + c] : 0.f;
        if constexpr (LATE) {
            // the tile's unigram level (shared by every row): uni, else <unk>,
            // else -1e30 (-> the floor); rows add their backoff sum
            float* lu = bias + 256;
            const float unk = isfinite(lm.unk_prob) ? static_cast<float>(lm.unk_prob) : -1e30f;
            for (int c = threadIdx.x; c < bnv; c += GEMM_THREADS) {
                const int col = n0 + c;
                float u = -1e30f;
                if (col < m.V) {
                    u = lm.uni[col];
                    if (isnan(u)) u = unk;
                }
                lu[c] = u;
            }
        }
        p.L = 0;
        p.acc_root = 0.f;
        if constexpr (LATE) {
            if (row < p.count) {
                double accd = 0.0;
                int c = st.lm_state[p.slot];
                while (c != 0 && p.L < kMaxOrder) {
                    p.chain[p.L] = c;
                    p.accs[p.L] = static_cast<float>(accd);
                    ++p.L;
                    accd += lm.backoff[c];
                    c = lm.suffix[c];
                }
                p.acc_root = static_cast<float>(accd);
            }
        }
        return p;
    }
    // probe q's column inside this chunk [col0, col0 + ntok): its logit
    __device__ __forceinline__ void write_probes(const Pre& pre, int slot, int col0, const float (&v)[8],
                                                 int ntok) const {
#pragma unroll
        for (int q = 0; q < PC; ++q) {
            const int d = pre.pc[q] - col0;
            if ((q < pre.npc) & (d >= 0) & (d < ntok)) {
                float x = v[0];
#pragma unroll
                for (int j = 1; j < 8; ++j) x = d == j ? v[j] : x;
                st.probe[static_cast<size_t>(slot) * cfg.K + q] = x;
            }
        }
    }
    template <class Acc>
    __device__ void run(uint32_t tmem, int grp, int lane, int m0, int nt, int n0, int bnv, int sb,
                        uint8_t* scratch, const Pre& pre, uint8_t* side, Acc acc) const {
        const bool tr = (st.trace & 1) && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0;
        long long tt = tr ? clock64() : 0;
        const int count = pre.count;
        const int r = grp * 32 + lane;
        const int row = m0 + r;
        const bool valid = row < count;
        const int slot = valid ? pre.slot : -1;
        const int ncols = m.R + m.ND;
        const int K = cfg.K;
        const int q = bnv >> 2;             // columns of this sub-block
        const int c_lo = sb * q;            // first tile column of the sub-block
        const int pitch = bnv + 1;
        float* lmt = reinterpret_cast<float*>(scratch);
        const float* bias = reinterpret_cast<const float*>(side);  // staged during the mainloop
        // late fusion LM row of this row / sub-block: the unigram level comes
        // from the tile's shared column table lu (+ the row's backoff sum); the
        // higher orders overwrite from shallow to deep (ngram_lm.cpp:363-416)
        // as sparse overrides: value in lmt, presence bit in ovm
        const float* lu = bias + 256;
        const float floor_v = static_cast<float>(kLogZeroFloor);
        const float acc_root = pre.acc_root;
        unsigned long long ovm = 0ull;
        if (LATE && valid) {
            const int L = pre.L;
            const int lo_tok = n0 + c_lo, hi_tok = min(n0 + c_lo + q, m.V);
            for (int l = L - 1; l >= 0; --l) {
                const int node = pre.chain[l];
                int lo = lm.cbeg[node], hi = lm.cend[node];
                const int end = hi;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (lm.etok[mid] < lo_tok) lo = mid + 1;
                    else hi = mid;
                }
                for (int e = lo; e < end; ++e) {
                    const int tk = lm.etok[e];
                    if (tk >= hi_tok) break;
                    const double p = lm.prob[lm.enode[e]];
                    if (!isnan(p)) {
                        lmt[r * pitch + (tk - n0)] = fmaxf(pre.accs[l] + static_cast<float>(p), floor_v);
                        ovm |= 1ull << (tk - lo_tok);
                    }
                }
            }
        }
        // LM value of tile column cc (of this thread's sub-block)
        auto lmval = [&](int cc) -> float {
            return ((ovm >> (cc - c_lo)) & 1ull) ? lmt[r * pitch + cc] : fmaxf(acc_root + lu[cc], floor_v);
        };
        __syncthreads();
        if (tr) {
            const long long t = clock64();
            g_gemm_trace[33] += t - tt;
            tt = t;
        }
        const float lamf = static_cast<float>(cfg.lam);
        float mx = -INFINITY, sm = 0.f;
        // no logit payload: with late fusion the logit is re-derived at the
        // staging as raw - lambda * lm (the LM value is re-read from the table)
        TopK<KM, false> top;
        constexpr float L2E = 1.4426950408889634f;
#ifndef TBEAM_EPI_PASSES
#define TBEAM_EPI_PASSES 1  // measurement: > 1 repeats the chunk loop (warm-code timing, trace slot 35)
#endif
        for (int pass = 0; pass < TBEAM_EPI_PASSES; ++pass) {
        if (pass == 1 && tr) {
            const long long t = clock64();
            g_gemm_trace[34] += t - tt;
            tt = t;
        }
        mx = -INFINITY;
        sm = 0.f;
        top.init();
        for (int c0 = c_lo; c0 < c_lo + q; c0 += 8) {
            float v[8];
            acc.ld8(tmem + c0, v);
            if (!valid) continue;
            const int col0 = n0 + c0;
            if (col0 + 8 <= m.V && c0 + 8 <= c_lo + q) {
                // interior chunk: 8 token columns, no predicates.  Online
                // log-sum-exp (exp2 with the scale folded into one FFMA), then
                // the top-K insert only when the chunk's best value enters.
                const float4 b0 = *reinterpret_cast<const float4*>(bias + c0);
                const float4 b1 = *reinterpret_cast<const float4*>(bias + c0 + 4);
                v[0] += b0.x; v[1] += b0.y; v[2] += b0.z; v[3] += b0.w;
                v[4] += b1.x; v[5] += b1.y; v[6] += b1.z; v[7] += b1.w;
                if (pre.npc) write_probes(pre, slot, col0, v, 8);
                const float cmax = fmaxf(fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3])),
                                         fmaxf(fmaxf(v[4], v[5]), fmaxf(v[6], v[7])));
                const float nm = fmaxf(mx, cmax);
                const float nmk = nm * L2E;
                float e[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) e[j] = exp2f(fmaf(v[j], L2E, -nmk));
                sm = sm * exp2f(fmaf(mx, L2E, -nmk)) + (((e[0] + e[1]) + (e[2] + e[3])) + ((e[4] + e[5]) + (e[6] + e[7])));
                mx = nm;
                float raw[8];
                float rmax = cmax;
                if constexpr (LATE) {
                    if (((ovm >> (c0 - c_lo)) & 0xFFull) == 0ull) {
                        const float4 u0 = *reinterpret_cast<const float4*>(lu + c0);
                        const float4 u1 = *reinterpret_cast<const float4*>(lu + c0 + 4);
                        const float uu[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
                        for (int j = 0; j < 8; ++j) raw[j] = fmaf(lamf, fmaxf(acc_root + uu[j], floor_v), v[j]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 8; ++j) raw[j] = fmaf(lamf, lmval(c0 + j), v[j]);
                    }
                    rmax = fmaxf(fmaxf(fmaxf(raw[0], raw[1]), fmaxf(raw[2], raw[3])),
                                 fmaxf(fmaxf(raw[4], raw[5]), fmaxf(raw[6], raw[7])));
                } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j) raw[j] = v[j];
                }
                // columns rise within a thread, so an equal value never
                // displaces a kept entry: "enters" is a strict compare
                if (rmax > top.v[KM - 1]) {
                    if constexpr (KM >= TBEAM_PUSH8_MIN) {
                        top.push8(raw, col0);
                    } else {
#pragma unroll
                        for (int j = 0; j < 8; ++j) top.push(raw[j], col0 + j, v[j]);
                    }
                }
                continue;
            }
            const int lim = min(8, min(c_lo + q, ncols - n0) - c0);  // live columns of the chunk
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = j < lim ? v[j] + bias[c0 + j] : -INFINITY;
            if (pre.npc) write_probes(pre, slot, col0, v, min(lim, m.V - col0));
            // online log-sum-exp over token + blank columns (trees, no chains)
            const int nstat = min(lim, m.V + 1 - col0);
            float t4[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                t4[j] = fmaxf(2 * j < nstat ? v[2 * j] : -INFINITY, 2 * j + 1 < nstat ? v[2 * j + 1] : -INFINITY);
            const float cmax = fmaxf(fmaxf(t4[0], t4[1]), fmaxf(t4[2], t4[3]));
            if (cmax > -INFINITY) {
                const float nm = fmaxf(mx, cmax);
                const float nmk = nm * L2E;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    t4[j] = (2 * j < nstat ? exp2f(fmaf(v[2 * j], L2E, -nmk)) : 0.f) +
                            (2 * j + 1 < nstat ? exp2f(fmaf(v[2 * j + 1], L2E, -nmk)) : 0.f);
                sm = sm * exp2f(fmaf(mx, L2E, -nmk)) + ((t4[0] + t4[1]) + (t4[2] + t4[3]));
                mx = nm;
            }
            const int ntok = min(lim, m.V - col0);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (j >= ntok && j < lim) {
                    const int col = col0 + j;
                    if (col == m.V) st.blank_logit[slot] = v[j];
                    else st.dur_logit[static_cast<size_t>(slot) * st.ndx + (col - m.R)] = v[j];
                }
            // top-K: every token column of the chunk through the insert
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (j < ntok) {
                    const float raw = LATE ? fmaf(lamf, lmval(c0 + j), v[j]) : v[j];
                    top.push(raw, col0 + j, v[j]);
                }
            }
        }
        }  // passes
        if (tr) {
            const long long t = clock64();
            g_gemm_trace[TBEAM_EPI_PASSES > 1 ? 35 : 34] += t - tt;
            tt = t;
        }
        // merge the four sub-block partials of each row inside the CTA: every
        // thread stages its sorted list in smem (the ring / LM table is free
        // by now), then the sub-block-0 thread of the row 4-way merges them
        // straight into the row's single partial record -- 4x fewer bytes and
        // merge lists for the select kernel.  Rows go in passes when 4 lists
        // of KM entries per row exceed the staging area.
        constexpr int SR = KM + 1;  // float4 records per staged list
        constexpr int RP = (160 * 1024) / (4 * SR * 16) >= 128 ? 128 : 64;
        float4* stage = reinterpret_cast<float4*>(scratch);
        // late fusion: the winners' LM values (fp32, as ranked) travel in the
        // record; read from the LM table before the staging overwrites it
        float lmq[LATE ? KM : 1];
        if constexpr (LATE) {
#pragma unroll
            for (int qq = 0; qq < KM; ++qq)
                lmq[qq] = (valid && top.ix[qq] != 0x7fffffff) ? lmval(top.ix[qq] - n0) : 0.f;
        }
        // (CLU: the row's CTA-level record goes to smem, after the staging
        // area, for the cluster merge below)
        float4* rec;
        if constexpr (CLU) {
            rec = reinterpret_cast<float4*>(scratch) + static_cast<size_t>(4 * SR) * RP + static_cast<size_t>(r) * SR;
        } else {
            const size_t pb = static_cast<size_t>(valid ? slot : 0) * st.NT + nt;
            rec = reinterpret_cast<float4*>(st.part + pb * part_stride(K));
        }
#pragma unroll 1
        for (int base = 0; base < 128; base += RP) {
            __syncthreads();  // LM-table reads / previous pass done
            const bool mine = r >= base && r < base + RP;
            if (mine) {
                float4* o = stage + (static_cast<size_t>(r - base) * 4 + sb) * SR;
                o[0] = make_float4(mx, sm, 0.f, 0.f);
#pragma unroll
                for (int qq = 0; qq < KM; ++qq) {
                    if (qq >= K) break;
                    float lq = 0.f;
                    if constexpr (LATE) lq = lmq[qq];
                    const float lgq = LATE ? top.v[qq] - lamf * lq : top.v[qq];
                    o[1 + qq] = make_float4(top.v[qq], __int_as_float(top.ix[qq]), lgq, lq);
                }
            }
            __syncthreads();
            if (mine && valid && sb == 0) {
                const float4* o = stage + static_cast<size_t>(r - base) * 4 * SR;
                float gm = -INFINITY;
#pragma unroll
                for (int l = 0; l < 4; ++l) gm = fmaxf(gm, o[l * SR].x);
                float gs = 0.f;
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    const float4 h = o[l * SR];
                    if (h.x > -INFINITY) gs += h.y * __expf(h.x - gm);
                }
                rec[0] = make_float4(gm, gs, 0.f, 0.f);
                int p0 = 1, p1 = 1, p2 = 1, p3 = 1;  // heads of the 4 lists
#pragma unroll 1
                for (int j = 0; j < K; ++j) {
                    const float4 h0 = p0 <= K ? o[0 * SR + p0] : make_float4(-INFINITY, __int_as_float(0x7fffffff), 0.f, 0.f);
                    const float4 h1 = p1 <= K ? o[1 * SR + p1] : make_float4(-INFINITY, __int_as_float(0x7fffffff), 0.f, 0.f);
                    const float4 h2 = p2 <= K ? o[2 * SR + p2] : make_float4(-INFINITY, __int_as_float(0x7fffffff), 0.f, 0.f);
                    const float4 h3 = p3 <= K ? o[3 * SR + p3] : make_float4(-INFINITY, __int_as_float(0x7fffffff), 0.f, 0.f);
                    float4 best = h0;
                    int w = 0;
                    auto better = [](const float4& x, const float4& y) {
                        const int xi = __float_as_int(x.y), yi = __float_as_int(y.y);
                        return (x.x > y.x) | ((x.x == y.x) & (xi < yi));
                    };
                    if (better(h1, best)) { best = h1; w = 1; }
                    if (better(h2, best)) { best = h2; w = 2; }
                    if (better(h3, best)) { best = h3; w = 3; }
                    const bool ok = __float_as_int(best.y) != 0x7fffffff;
                    rec[1 + j] = make_float4(best.x, __int_as_float(ok ? __float_as_int(best.y) : -1), best.z, best.w);
                    p0 += w == 0;
                    p1 += w == 1;
                    p2 += w == 2;
                    p3 += w == 3;
                }
            }
        }
        if constexpr (CLU) cluster_merge(reinterpret_cast<float4*>(scratch) + static_cast<size_t>(4 * SR) * RP, m0,
                                         nt, count);
    }

    // CLU: CTA rank cr of the cluster merges rows [cr*128/CL, (cr+1)*128/CL):
    // one warp per row, lane l < CL reads CTA l's record of the row through
    // DSMEM; (max, sum-exp) combine by log-sum-exp, the K entries by a
    // CL-way merge of the sorted lists (value desc, column asc).
    __device__ __forceinline__ void cluster_merge(const float4* crec, int m0, int nt, int count) const {
        constexpr int SR = KM + 1;
        namespace cg = cooperative_groups;
        cg::cluster_group cluster = cg::this_cluster();
        cluster.sync();  // every CTA's records are in its smem
        const int CL = static_cast<int>(cluster.dim_blocks().y);
        const int cr = static_cast<int>(cluster.block_rank());
        const int ci = nt / CL;
        const int rpc = 128 / CL;
        const int warp = threadIdx.x >> 5, ln = threadIdx.x & 31;
        const int K = cfg.K;
        for (int rr = warp; rr < rpc; rr += GEMM_THREADS / 32) {
            const int r2 = cr * rpc + rr;
            const int row2 = m0 + r2;
            if (row2 >= count) break;  // (warp-uniform; later rows are past the count too)
            const int slot2 = st.act_list[par * st.S + row2];
            float4* out = reinterpret_cast<float4*>(st.part + (static_cast<size_t>(slot2) * st.NT + ci) *
                                                                  part_stride(K));
            const float4* src = ln < CL ? cluster.map_shared_rank(crec + static_cast<size_t>(r2) * SR, ln) : crec;
            const float4 h = ln < CL ? src[0] : make_float4(-INFINITY, 0.f, 0.f, 0.f);
            float gm = h.x;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, o));
            float gs = (h.x > -INFINITY) ? h.y * __expf(h.x - gm) : 0.f;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) gs += __shfl_xor_sync(0xffffffffu, gs, o);
            if (ln == 0) out[0] = make_float4(gm, gs, 0.f, 0.f);
            int pos = 1;
            auto load = [&](int q) {
                float4 e = make_float4(-INFINITY, __int_as_float(0x7fffffff), 0.f, 0.f);
                if (ln < CL && q <= K) {
                    e = src[q];
                    if (__float_as_int(e.y) < 0) e = make_float4(-INFINITY, __int_as_float(0x7fffffff), 0.f, 0.f);
                }
                return e;
            };
            float4 cur = load(pos);
#pragma unroll 1
            for (int j = 0; j < K; ++j) {
                float bv = cur.x;
                int bi = __float_as_int(cur.y), bl = ln;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
                    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                    const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
                    const bool take = (ov > bv) | ((ov == bv) & ((oi < bi) | ((oi == bi) & (ol < bl))));
                    bv = take ? ov : bv;
                    bi = take ? oi : bi;
                    bl = take ? ol : bl;
                }
                if (ln == bl) {
                    const bool ok = bi != 0x7fffffff;
                    out[1 + j] = ok ? cur : make_float4(-INFINITY, __int_as_float(-1), 0.f, 0.f);
                    ++pos;
                    cur = load(pos);
                }
            }
        }
        cluster.sync();  // no CTA leaves while a peer may still read its records
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
    __device__ int tl_round() const { return -1; }
    __device__ void finish() const {}
    struct Pre {};
    __device__ Pre prefetch(int, int, int, int, int, int, uint8_t*) const { return Pre{}; }
    template <class Acc>
    __device__ void run(uint32_t tmem, int grp, int lane, int m0, int nt, int n0, int bnv, int sb, uint8_t*,
                        const Pre&, uint8_t*, Acc acc) const {
        const int row = m0 + grp * 32 + lane;
        const bool valid = row < nrows;
        float* out = st.encp + static_cast<size_t>(row) * m.J;
        const int q = bnv >> 2;
        for (int c0 = sb * q; c0 < sb * q + q; c0 += 8) {
            float v[8];
            acc.ld8(tmem + c0, v);
            if (!valid) continue;
            const int col = n0 + c0;
            if (col + 8 <= m.J) {
                const float4 b0 = __ldg(reinterpret_cast<const float4*>(m.b_enc + col));
                const float4 b1 = __ldg(reinterpret_cast<const float4*>(m.b_enc + col) + 1);
                reinterpret_cast<float4*>(out + col)[0] = make_float4(v[0] + b0.x, v[1] + b0.y, v[2] + b0.z, v[3] + b0.w);
                reinterpret_cast<float4*>(out + col)[1] = make_float4(v[4] + b1.x, v[5] + b1.y, v[6] + b1.z, v[7] + b1.w);
            } else {
                for (int j = 0; j < 8 && col + j < m.J; ++j) out[col + j] = v[j] + m.b_enc[col + j];
            }
        }
    }
};

// ---------------------------------------------------------------------------
// LSTM gates epilogue: tile nt = hidden units [32nt, 32nt+32) x (i,f,g,o);
// sub-block sb = units [32nt + 8sb, +8)
// ---------------------------------------------------------------------------
struct GatesEpi {
    static constexpr int kTrace = 1;
    DevModel m;
    DevState st;
    int par;
    __device__ int rows() const { return st.upd_count[par]; }
    __device__ int tl_round() const { return *st.g - (st.round_in_proj ? 0 : 1); }
    __device__ void finish() const {}
    // issued during the mainloop: the row's pool entries / token, then its
    // input-table slice and parent cell state
    struct Pre {
        int count;
        int dst;
        float4 xv[4][2], cv[2];
    };
    __device__ Pre prefetch(int grp, int lane, int m0, int n0, int bnv, int sb, uint8_t*) const {
        Pre p;
        const int row = m0 + grp * 32 + lane;
        p.count = st.upd_count[par];
        p.dst = 0;
        if (row < p.count) {
            const size_t S = st.S;
            const int H = m.H;
            const size_t src = st.upd_src[par * S + row];
            p.dst = st.upd_dst[par * S + row];
            const int tok = st.upd_tok[par * S + row];
            const int u0 = blockIdx.y * 32 + 8 * sb;
            const float* __restrict__ x = m.xtab + static_cast<size_t>(tok) * 4 * H + u0;
#pragma unroll
            for (int g = 0; g < 4; ++g)
#pragma unroll
                for (int h = 0; h < 2; ++h) p.xv[g][h] = __ldg(reinterpret_cast<const float4*>(x + g * H) + h);
            const float4* cp = reinterpret_cast<const float4*>(st.c + src * H + u0);
            p.cv[0] = cp[0];
            p.cv[1] = cp[1];
        }
        return p;
    }
    template <class Acc>
    __device__ void run(uint32_t tmem, int grp, int lane, int m0, int nt, int n0, int bnv, int sb, uint8_t*,
                        const Pre& pre, uint8_t*, Acc acc) const {
        const int row = m0 + grp * 32 + lane;
        const bool valid = row < pre.count;
        float gi[8], gf[8], gg[8], go[8];
        acc.ld8(tmem + 8 * sb, gi);
        acc.ld8(tmem + 32 + 8 * sb, gf);
        acc.ld8(tmem + 64 + 8 * sb, gg);
        acc.ld8(tmem + 96 + 8 * sb, go);
        if (!valid) return;
        const int H = m.H;
        const size_t dst = pre.dst;
        const int u0 = nt * 32 + 8 * sb;
        float4* __restrict__ cn = reinterpret_cast<float4*>(st.c + dst * H + u0);
        float4* __restrict__ hn = reinterpret_cast<float4*>(st.h + dst * H + u0);
        uint2* __restrict__ hb = reinterpret_cast<uint2*>(st.hB16 + static_cast<size_t>(row) * st.Hp + u0);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float xa[4][4] = {{pre.xv[0][h].x, pre.xv[0][h].y, pre.xv[0][h].z, pre.xv[0][h].w},
                                    {pre.xv[1][h].x, pre.xv[1][h].y, pre.xv[1][h].z, pre.xv[1][h].w},
                                    {pre.xv[2][h].x, pre.xv[2][h].y, pre.xv[2][h].z, pre.xv[2][h].w},
                                    {pre.xv[3][h].x, pre.xv[3][h].y, pre.xv[3][h].z, pre.xv[3][h].w}};
            const float ca[4] = {pre.cv[h].x, pre.cv[h].y, pre.cv[h].z, pre.cv[h].w};
            float cn4[4], hn4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int u = h * 4 + e;
                const float ig = __fdividef(1.f, 1.f + __expf(-(gi[u] + xa[0][e])));
                const float fg = __fdividef(1.f, 1.f + __expf(-(gf[u] + xa[1][e])));
                const float g = tanhf(gg[u] + xa[2][e]);
                const float og = __fdividef(1.f, 1.f + __expf(-(go[u] + xa[3][e])));
                cn4[e] = fg * ca[e] + ig * g;
                hn4[e] = og * tanhf(cn4[e]);
            }
            cn[h] = make_float4(cn4[0], cn4[1], cn4[2], cn4[3]);
            hn[h] = make_float4(hn4[0], hn4[1], hn4[2], hn4[3]);
            const __nv_bfloat162 h01 = __floats2bfloat162_rn(hn4[0], hn4[1]);
            const __nv_bfloat162 h23 = __floats2bfloat162_rn(hn4[2], hn4[3]);
            uint2 pk;
            pk.x = *reinterpret_cast<const uint32_t*>(&h01);
            pk.y = *reinterpret_cast<const uint32_t*>(&h23);
            hb[h] = pk;
        }
    }
};

// ---------------------------------------------------------------------------
// LSTM gates epilogue, 8-unit tiles (full-K GEMM): tile nt = hidden units
// [8nt, 8nt+8) x (i,f,g,o) = 32 columns; sub-block 0 of each row does the cell
// ---------------------------------------------------------------------------
// EXACT (precision fp32 on the tensor cores): accurate expf / division, like
// the CUDA-core cell (kernels_simt.cu), and h' staged as three bf16 planes
template <bool EXACT>
struct GatesEpi8T {
    static constexpr int kTrace = 1;
    DevModel m;
    DevState st;
    int par;
    __device__ int rows() const { return st.upd_count[par]; }
    __device__ int tl_round() const { return *st.g - (st.round_in_proj ? 0 : 1); }
    __device__ void finish() const {}
    struct Pre {
        int count;
        int dst;
        float4 xv[4][2], cv[2];
    };
    __device__ Pre prefetch(int grp, int lane, int m0, int n0, int bnv, int sb, uint8_t*) const {
        Pre p;
        const int row = m0 + grp * 32 + lane;
        p.count = st.upd_count[par];
        p.dst = 0;
        if (sb == 0 && row < p.count) {
            const size_t S = st.S;
            const int H = m.H;
            const size_t src = st.upd_src[par * S + row];
            p.dst = st.upd_dst[par * S + row];
            const int tok = st.upd_tok[par * S + row];
            const int u0 = n0 / 4;  // tile = 8 units x 4 gates = 32 columns
            const float* __restrict__ x = m.xtab + static_cast<size_t>(tok) * 4 * H + u0;
#pragma unroll
            for (int g = 0; g < 4; ++g)
#pragma unroll
                for (int h = 0; h < 2; ++h) p.xv[g][h] = __ldg(reinterpret_cast<const float4*>(x + g * H) + h);
            const float4* cp = reinterpret_cast<const float4*>(st.c + src * H + u0);
            p.cv[0] = cp[0];
            p.cv[1] = cp[1];
        }
        return p;
    }
    template <class Acc>
    __device__ void run(uint32_t tmem, int grp, int lane, int m0, int nt, int n0, int bnv, int sb, uint8_t*,
                        const Pre& pre, uint8_t*, Acc acc) const {
        if (sb != 0) return;  // (warp-uniform) one warp per row group does the cell
        const int row = m0 + grp * 32 + lane;
        const bool valid = row < pre.count;
        float gi[8], gf[8], gg[8], go[8];
        acc.ld8(tmem, gi);
        acc.ld8(tmem + 8, gf);
        acc.ld8(tmem + 16, gg);
        acc.ld8(tmem + 24, go);
        if (!valid) return;
        const int H = m.H;
        const size_t dst = pre.dst;
        const int u0 = nt * 8;
        float4* __restrict__ cn = reinterpret_cast<float4*>(st.c + dst * H + u0);
        float4* __restrict__ hn = reinterpret_cast<float4*>(st.h + dst * H + u0);
        uint4 hb16;
        uint32_t* hbw = reinterpret_cast<uint32_t*>(&hb16);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float xa[4][4] = {{pre.xv[0][h].x, pre.xv[0][h].y, pre.xv[0][h].z, pre.xv[0][h].w},
                                    {pre.xv[1][h].x, pre.xv[1][h].y, pre.xv[1][h].z, pre.xv[1][h].w},
                                    {pre.xv[2][h].x, pre.xv[2][h].y, pre.xv[2][h].z, pre.xv[2][h].w},
                                    {pre.xv[3][h].x, pre.xv[3][h].y, pre.xv[3][h].z, pre.xv[3][h].w}};
            const float ca[4] = {pre.cv[h].x, pre.cv[h].y, pre.cv[h].z, pre.cv[h].w};
            float cn4[4], hn4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int u = h * 4 + e;
                float ig, fg, og;
                if constexpr (EXACT) {
                    ig = 1.f / (1.f + expf(-(gi[u] + xa[0][e])));
                    fg = 1.f / (1.f + expf(-(gf[u] + xa[1][e])));
                    og = 1.f / (1.f + expf(-(go[u] + xa[3][e])));
                } else {
                    ig = __fdividef(1.f, 1.f + __expf(-(gi[u] + xa[0][e])));
                    fg = __fdividef(1.f, 1.f + __expf(-(gf[u] + xa[1][e])));
                    og = __fdividef(1.f, 1.f + __expf(-(go[u] + xa[3][e])));
                }
                const float g = tanhf(gg[u] + xa[2][e]);
                cn4[e] = fg * ca[e] + ig * g;
                hn4[e] = og * tanhf(cn4[e]);
            }
            cn[h] = make_float4(cn4[0], cn4[1], cn4[2], cn4[3]);
            hn[h] = make_float4(hn4[0], hn4[1], hn4[2], hn4[3]);
            if constexpr (EXACT) {
                put_op4(st.hB16 + static_cast<size_t>(row) * st.Hp + u0 + 4 * h, st.hpl, 1, hn4[0], hn4[1], hn4[2],
                        hn4[3]);
            } else {
                const __nv_bfloat162 h01 = __floats2bfloat162_rn(hn4[0], hn4[1]);
                const __nv_bfloat162 h23 = __floats2bfloat162_rn(hn4[2], hn4[3]);
                hbw[2 * h] = *reinterpret_cast<const uint32_t*>(&h01);
                hbw[2 * h + 1] = *reinterpret_cast<const uint32_t*>(&h23);
            }
        }
        if constexpr (!EXACT) *reinterpret_cast<uint4*>(st.hB16 + static_cast<size_t>(row) * st.Hp + u0) = hb16;
    }
};
using GatesEpi8 = GatesEpi8T<false>;

// ---------------------------------------------------------------------------
// LSTM gates, 12-unit tiles (N = 48 = 12 units x (i,f,g,o)): ceil(H/12) tiles,
// so two M-tiles of token rows (<= 256, the beam's usual count) are 108 CTAs
// -- one wave on 148 SMs at one 223-KB CTA per SM (8-unit tiles need 160
// CTAs: the second wave's CTAs wait for the first wave's exits, ~5 us of
// release skew per round).  The cell runs on all four epilogue sub-blocks,
// three units per thread (the 8-unit epilogue uses one sub-block).
// Opt-in (TBEAM_GATES12=1): measured SLOWER at the bench shape -- busy 6.9 ->
// 11.2 us per launch (skew 6.0 -> 3.2 us): the 223-KB CTA's operand boxes and
// the scalar x / c / h accesses of the 3-unit slices cost more than the wave.
// Weights: row t*48 + gate*12 + u <- W_hh row gate*H + 12t + u (zero rows past H).
// ---------------------------------------------------------------------------
struct GatesEpi12 {
    static constexpr int kTrace = 1;
    static constexpr int U = 12, US = 3;  // units per tile, per sub-block
    DevModel m;
    DevState st;
    int par;
    __device__ int rows() const { return st.upd_count[par]; }
    __device__ int tl_round() const { return *st.g - (st.round_in_proj ? 0 : 1); }
    __device__ void finish() const {}
    struct Pre {
        int count, dst;
        float x[4][US], c[US];
    };
    __device__ Pre prefetch(int grp, int lane, int m0, int n0, int bnv, int sb, uint8_t*) const {
        Pre p;
        const int row = m0 + grp * 32 + lane;
        p.count = st.upd_count[par];
        p.dst = 0;
        const int H = m.H;
        const int u0 = (n0 / 48) * U + sb * US;
        if (row < p.count) {
            const size_t S = st.S;
            const size_t src = st.upd_src[par * S + row];
            p.dst = st.upd_dst[par * S + row];
            const int tok = st.upd_tok[par * S + row];
            const float* __restrict__ x = m.xtab + static_cast<size_t>(tok) * 4 * H;
#pragma unroll
            for (int e = 0; e < US; ++e) {
                const int u = min(u0 + e, H - 1);
#pragma unroll
                for (int g = 0; g < 4; ++g) p.x[g][e] = __ldg(x + g * H + u);
                p.c[e] = st.c[src * H + u];
            }
        }
        return p;
    }
    template <class Acc>
    __device__ void run(uint32_t tmem, int grp, int lane, int m0, int nt, int n0, int bnv, int sb, uint8_t*,
                        const Pre& pre, uint8_t*, Acc acc) const {
        const int row = m0 + grp * 32 + lane;
        // gate g of this sub-block's units: columns g*12 + 3*sb + e, inside
        // the two 8-column loads from the 8-aligned column below them
        float gv[4][US];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const int c0 = g * U + sb * US;
            const int base = c0 & ~7;
            float v[16];
            acc.ld8(tmem + base, *reinterpret_cast<float(*)[8]>(v));
            acc.ld8(tmem + base + 8, *reinterpret_cast<float(*)[8]>(v + 8));
#pragma unroll
            for (int e = 0; e < US; ++e) gv[g][e] = v[c0 - base + e];
        }
        if (row >= pre.count) return;
        const int H = m.H;
        const size_t dst = pre.dst;
        const int u0 = nt * U + sb * US;
#pragma unroll
        for (int e = 0; e < US; ++e) {
            const int u = u0 + e;
            if (u >= H) break;
            const float ig = __fdividef(1.f, 1.f + __expf(-(gv[0][e] + pre.x[0][e])));
            const float fg = __fdividef(1.f, 1.f + __expf(-(gv[1][e] + pre.x[1][e])));
            const float g = tanhf(gv[2][e] + pre.x[2][e]);
            const float og = __fdividef(1.f, 1.f + __expf(-(gv[3][e] + pre.x[3][e])));
            const float cn = fg * pre.c[e] + ig * g;
            const float hn = og * tanhf(cn);
            st.c[dst * H + u] = cn;
            st.h[dst * H + u] = hn;
            st.hB16[static_cast<size_t>(row) * st.Hp + u] = __float2bfloat16_rn(hn);
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
    cudaGraphConditionalHandle hcond;
    int set_cond;
    __device__ int rows() const { return st.upd_count[par]; }
    __device__ int tl_round() const { return *st.g - (st.round_in_proj ? 0 : 1); }
    // the round's last kernel closes it (st.round_in_proj): round counter and
    // the CUDA-graph WHILE condition "a stream is still decoding"
    __device__ void finish() const {
        if (!st.round_in_proj) return;
        const int rounds = *st.g + (*st.live ? 1 : 0);
        *st.g = rounds;
        if (set_cond) cudaGraphSetConditional(hcond, (*st.n_done < st.B && rounds < st.max_cols) ? 1u : 0u);
    }
    // issued during the mainloop: the row's slot, pool entry, next-round
    // operand row, and the encoder-projection / bias slices it combines with
    struct Pre {
        int count, pos, dst;
        float4 e[2], bq[2];
    };
    __device__ Pre prefetch(int grp, int lane, int m0, int n0, int bnv, int sb, uint8_t*) const {
        Pre p;
        const int row = m0 + grp * 32 + lane;
        p.count = st.upd_count[par];
        p.pos = -1;
        p.dst = 0;
        const int col0 = n0 + sb * (bnv >> 2);
        if (row < p.count) {
            const size_t S = st.S;
            const int slot = st.upd_list[par * S + row];
            p.dst = st.upd_dst[par * S + row];
            p.pos = st.act_pos[slot];
            const int b = slot / st.K;
            if (col0 + 8 <= m.J) {
                const float* ep = st.encp + (static_cast<size_t>(b) * st.Tmax + min(st.t[b], st.Tmax - 1)) * m.J;
                p.e[0] = reinterpret_cast<const float4*>(ep + col0)[0];
                p.e[1] = reinterpret_cast<const float4*>(ep + col0)[1];
                p.bq[0] = __ldg(reinterpret_cast<const float4*>(m.b_pred + col0));
                p.bq[1] = __ldg(reinterpret_cast<const float4*>(m.b_pred + col0) + 1);
            }
        }
        return p;
    }
    template <class Acc>
    __device__ void run(uint32_t tmem, int grp, int lane, int m0, int nt, int n0, int bnv, int sb, uint8_t*,
                        const Pre& pre, uint8_t*, Acc acc) const {
        const int row = m0 + grp * 32 + lane;
        const bool valid = row < pre.count;
        const int q = bnv >> 2;
        float v[8];
        acc.ld8(tmem + sb * q, v);  // bnv = 32 -> one chunk of 8 per sub-block
        if (!valid) return;
        const int pos = pre.pos;
        float* pd = st.pred + static_cast<size_t>(pre.dst) * m.J;
        const int col0 = n0 + sb * q;
        if (col0 + 8 <= m.J) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float4 bq = pre.bq[h];
                const float4 p = make_float4(v[4 * h] + bq.x, v[4 * h + 1] + bq.y, v[4 * h + 2] + bq.z,
                                             v[4 * h + 3] + bq.w);
                reinterpret_cast<float4*>(pd + col0)[h] = p;
                if (pos >= 0) {
                    const float4 e = pre.e[h];
                    put_op4(st.z16 + static_cast<size_t>(pos) * st.Jp + col0 + 4 * h, st.zpl, st.split3,
                            tanhf(e.x + p.x), tanhf(e.y + p.y), tanhf(e.z + p.z), tanhf(e.w + p.w));
                }
            }
        } else {
            const int slot = st.upd_list[par * st.S + row];
            const int b = slot / st.K;
            const float* ep = st.encp + (static_cast<size_t>(b) * st.Tmax + min(st.t[b], st.Tmax - 1)) * m.J;
            for (int j = 0; j < 8 && col0 + j < m.J; ++j) {
                const float p = v[j] + m.b_pred[col0 + j];
                pd[col0 + j] = p;
                if (pos >= 0)
                    put_op(st.z16 + static_cast<size_t>(pos) * st.Jp + col0 + j, st.zpl, st.split3, tanhf(ep[col0 + j] + p));
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

template <int BN, class Epi, int MC = 1>
void launch_gemm(const TcMap& a, const TcMap& b, int K, int bnv, int m_tiles, int n_tiles, const Epi& epi,
                 cudaStream_t s, int cluster_n = 1) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(m_tiles, n_tiles);
    lc.blockDim = dim3(GEMM_THREADS);
    lc.dynamicSmemBytes = tc_smem_bytes<BN>();
    lc.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = 1;
    at[1].val.clusterDim.y = MC > 1 ? MC : cluster_n;
    at[1].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = (MC > 1 || cluster_n > 1) ? 2 : 1;
    cudaLaunchKernelEx(&lc, tc_gemm<BN, Epi, MC>, a.map, b.map, K, bnv, epi);
}

template <int BN, class Epi>
void launch_fk(const TcMap* a3, const TcMap& b, int nk, int bnv, int m_tiles, int n_tiles, const Epi& epi,
               cudaStream_t s) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(n_tiles, m_tiles);
    lc.blockDim = dim3(GEMM_THREADS);
    lc.dynamicSmemBytes = fk_smem_bytes<BN>();
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    cudaLaunchKernelEx(&lc, tc_gemm_fk<BN, Epi>, a3[0].map, a3[1].map, a3[2].map, b.map, nk, bnv, epi);
}

template <class Epi>
void launch_s3(const TcMap* a3, const TcMap& b, int nk, int per, int ks, int clu, int m_tiles, int n_tiles,
               const Epi& epi, cudaStream_t s) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(n_tiles, m_tiles, ks);
    lc.blockDim = dim3(GEMM_THREADS);
    lc.dynamicSmemBytes = s3_smem_bytes();
    lc.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = 1;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = ks;
    lc.attrs = at;
    clu = clu && ks > 1;
    lc.numAttrs = clu ? 2 : 1;
    cudaLaunchKernelEx(&lc, tc_gemm_s3<Epi>, a3[0].map, a3[1].map, a3[2].map, b.map, nk, per, clu, epi);
}

template <class Epi>
void set_s3_attr() {
    cudaFuncSetAttribute(tc_gemm_s3<Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize, s3_smem_bytes());
}

template <int BN, class Epi>
void set_fk_attr() {
    cudaFuncSetAttribute(tc_gemm_fk<BN, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize, fk_smem_bytes<BN>());
}

template <int BN, class Epi, int MC = 1>
void set_smem_attr() {
    cudaFuncSetAttribute(tc_gemm<BN, Epi, MC>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem_bytes<BN>());
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

TcMap make_tc_map3(const void* base, int rows, int nk, int pitch_elems, int box_rows, int depth) {
    load_encode();
    TcMap t{};
    cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(nk)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(pitch_elems) * 2, 128};
    cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(depth > 0 ? depth : nk)};
    cuuint32_t es[3] = {1, 1, 1};
    const CUresult r = g_encode(&t.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                                box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (3-D) failed: " + std::to_string(r));
    return t;
}

TcMap make_tc_map4(const void* base, int rows, int nk, int pitch_elems, size_t plane_elems, int box_rows, int depth) {
    load_encode();
    TcMap t{};
    cuuint64_t dims[4] = {64, static_cast<cuuint64_t>(rows), 3, static_cast<cuuint64_t>(nk)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(pitch_elems) * 2, static_cast<cuuint64_t>(plane_elems) * 2, 128};
    cuuint32_t box[4] = {64, static_cast<cuuint32_t>(box_rows), 3, static_cast<cuuint32_t>(depth)};
    cuuint32_t es[4] = {1, 1, 1, 1};
    const CUresult r = g_encode(&t.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
                                box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (4-D) failed: " + std::to_string(r));
    return t;
}

int fk_abox_depth(int nk) { return (nk + FK_ABOXES - 1) / FK_ABOXES; }

int tc_stages_for(int bn) {
    return bn == 32 ? tc_stages<32>() : bn == 64 ? tc_stages<64>() : bn == 128 ? tc_stages<128>() : tc_stages<256>();
}

void tl_read_tc(int enable, unsigned long long* out) {
    if (out) cudaMemcpyFromSymbol(out, g_tl_tc, sizeof(unsigned long long) * kTlRounds * 16);
    std::vector<unsigned long long> init(static_cast<size_t>(kTlRounds) * 16);
    for (size_t i = 0; i < init.size(); ++i) init[i] = (i % 4 == 0 || i % 4 == 1) ? ~0ull : 0ull;
    cudaMemcpyToSymbol(g_tl_tc, init.data(), init.size() * sizeof(unsigned long long));
}

void gemm_trace(int enable, long long* out) {
    if (out) {
        cudaMemcpyFromSymbol(out, g_gemm_trace, sizeof(long long) * 40);
    }
    long long z[40] = {};
    cudaMemcpyToSymbol(g_gemm_trace, z, sizeof(z));
}

void configure_tc_kernels() {
    set_smem_attr<32, ProjEpi, 4>();
#define TBEAM_JOINT_ATTR(BNV)                                                                         \
    set_smem_attr<BNV, JointEpi<1, false>>();                                                         \
    set_smem_attr<BNV, JointEpi<4, false>>();                                                         \
    set_smem_attr<BNV, JointEpi<8, false>>();                                                         \
    set_smem_attr<BNV, JointEpi<16, false>>();                                                        \
    set_smem_attr<BNV, JointEpi<32, false>>();                                                        \
    set_smem_attr<BNV, JointEpi<1, true>>();                                                          \
    set_smem_attr<BNV, JointEpi<4, true>>();                                                          \
    set_smem_attr<BNV, JointEpi<8, true>>();                                                          \
    set_smem_attr<BNV, JointEpi<16, true>>();                                                         \
    set_smem_attr<BNV, JointEpi<32, true>>()
    TBEAM_JOINT_ATTR(32);
    TBEAM_JOINT_ATTR(64);
    TBEAM_JOINT_ATTR(256);
#undef TBEAM_JOINT_ATTR
    set_smem_attr<64, JointEpi<8, false, true>>();
    set_smem_attr<64, JointEpi<8, true, true>>();
    set_smem_attr<64, JointEpi<16, false, true>>();
    set_smem_attr<64, JointEpi<16, true, true>>();
    set_smem_attr<256, JointEpi<8, false, true>>();
    set_smem_attr<256, JointEpi<8, true, true>>();
    set_smem_attr<256, JointEpi<16, false, true>>();
    set_smem_attr<256, JointEpi<16, true, true>>();
    set_fk_attr<32, JointEpi<1, false>>();
    set_fk_attr<32, JointEpi<4, false>>();
    set_fk_attr<32, JointEpi<8, false>>();
    set_fk_attr<32, JointEpi<16, false>>();
    set_fk_attr<32, JointEpi<32, false>>();
    set_fk_attr<32, JointEpi<1, true>>();
    set_fk_attr<32, JointEpi<4, true>>();
    set_fk_attr<32, JointEpi<8, true>>();
    set_fk_attr<32, JointEpi<16, true>>();
    set_fk_attr<32, JointEpi<32, true>>();
    set_fk_attr<32, GatesEpi8>();
    set_fk_attr<48, GatesEpi12>();
    set_fk_attr<32, ProjEpi>();
    set_smem_attr<128, EncProjEpi>();
    set_smem_attr<128, GatesEpi>();
    set_smem_attr<32, ProjEpi>();
    set_s3_attr<JointEpi<1, false>>();
    set_s3_attr<JointEpi<4, false>>();
    set_s3_attr<JointEpi<8, false>>();
    set_s3_attr<JointEpi<16, false>>();
    set_s3_attr<JointEpi<32, false>>();
    set_s3_attr<JointEpi<1, true>>();
    set_s3_attr<JointEpi<4, true>>();
    set_s3_attr<JointEpi<8, true>>();
    set_s3_attr<JointEpi<16, true>>();
    set_s3_attr<JointEpi<32, true>>();
    set_s3_attr<GatesEpi8T<true>>();
    set_s3_attr<ProjEpi>();
}

void launch_joint_tc(const DevModel& m, const DevLm& lm, const DevCfg& cfg, const DevState& st, const TcPlan& p,
                     int par, cudaStream_t s) {
    const int m_tiles = (st.S + BM - 1) / BM;
    const int K = cfg.K;
#define TBEAM_JOINT_L(BNV, KMV, LT)                                                                   \
    launch_gemm<BNV, JointEpi<KMV, LT>>(p.z, p.wout, m.J, p.joint_bnv, m_tiles, p.joint_nt,         \
                                        JointEpi<KMV, LT>{m, lm, cfg, st, par}, s)
#define TBEAM_JOINT(BNV, KMV)                                                                         \
    do {                                                                                              \
        if (cfg.late) TBEAM_JOINT_L(BNV, KMV, true);                                                  \
        else TBEAM_JOINT_L(BNV, KMV, false);                                                          \
    } while (0)
#define TBEAM_JOINT_FK(KMV)                                                                           \
    do {                                                                                              \
        if (cfg.late)                                                                                 \
            launch_fk<32, JointEpi<KMV, true>>(p.zA, p.wout3, p.nk_j, p.joint_bnv, m_tiles, p.joint_nt, \
                                               JointEpi<KMV, true>{m, lm, cfg, st, par}, s);          \
        else                                                                                          \
            launch_fk<32, JointEpi<KMV, false>>(p.zA, p.wout3, p.nk_j, p.joint_bnv, m_tiles, p.joint_nt, \
                                                JointEpi<KMV, false>{m, lm, cfg, st, par}, s);        \
    } while (0)
#define TBEAM_JOINT_S3(KMV)                                                                           \
    do {                                                                                              \
        if (cfg.late)                                                                                 \
            launch_s3(p.zS, p.woutS, p.nk_j, p.s3_per_j, p.s3_ks_j, p.s3_clu, m_tiles, p.joint_nt,       \
                      JointEpi<KMV, true>{m, lm, cfg, st, par}, s);                                   \
        else                                                                                          \
            launch_s3(p.zS, p.woutS, p.nk_j, p.s3_per_j, p.s3_ks_j, p.s3_clu, m_tiles, p.joint_nt,       \
                      JointEpi<KMV, false>{m, lm, cfg, st, par}, s);                                  \
    } while (0)
    if (p.s3) {
        if (K <= 1) TBEAM_JOINT_S3(1);
        else if (K <= 4) TBEAM_JOINT_S3(4);
        else if (K <= 8) TBEAM_JOINT_S3(8);
        else if (K <= 16) TBEAM_JOINT_S3(16);
        else TBEAM_JOINT_S3(32);
    } else if (p.fk_joint) {
        if (K <= 1) TBEAM_JOINT_FK(1);
        else if (K <= 4) TBEAM_JOINT_FK(4);
        else if (K <= 8) TBEAM_JOINT_FK(8);
        else if (K <= 16) TBEAM_JOINT_FK(16);
        else TBEAM_JOINT_FK(32);
    } else if (p.joint_cl > 1) {  // cluster-merged tile lists (K 5..16, BN 64 / 256)
#define TBEAM_JOINT_C(BNV, KMV)                                                                       \
    do {                                                                                              \
        if (cfg.late)                                                                                 \
            launch_gemm<BNV, JointEpi<KMV, true, true>>(p.z, p.wout, m.J, p.joint_bnv, m_tiles, p.joint_nt, \
                                                        JointEpi<KMV, true, true>{m, lm, cfg, st, par}, s, \
                                                        p.joint_cl);                                  \
        else                                                                                          \
            launch_gemm<BNV, JointEpi<KMV, false, true>>(p.z, p.wout, m.J, p.joint_bnv, m_tiles, p.joint_nt, \
                                                         JointEpi<KMV, false, true>{m, lm, cfg, st, par}, s, \
                                                         p.joint_cl);                                 \
    } while (0)
        if (p.joint_bn == 64) {
            if (K <= 8) TBEAM_JOINT_C(64, 8);
            else TBEAM_JOINT_C(64, 16);
        } else {
            if (K <= 8) TBEAM_JOINT_C(256, 8);
            else TBEAM_JOINT_C(256, 16);
        }
#undef TBEAM_JOINT_C
    } else if (p.joint_bn == 32) {
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
#undef TBEAM_JOINT_L
#undef TBEAM_JOINT_FK
#undef TBEAM_JOINT_S3

}

void launch_encproj_tc(const DevModel& m, const DevState& st, const TcPlan& p, int rows, cudaStream_t s) {
    const int m_tiles = (rows + BM - 1) / BM;
    const int n_tiles = (m.J + 127) / 128;
    launch_gemm<128, EncProjEpi>(p.enc, p.wenc, m.D, 128, m_tiles, n_tiles, EncProjEpi{m, st, rows}, s);
}

void launch_lstm_tc(const DevModel& m, const DevState& st, const TcPlan& p, int par, cudaGraphConditionalHandle h,
                    int set_cond, cudaStream_t s, int part) {
    const int m_tiles = (st.S + BM - 1) / BM;
    if (p.s3) {
        if (part != 1)
            launch_s3(p.hAS, p.whhS, p.nk_h, p.s3_per_h, p.s3_ks_h, p.s3_clu, m_tiles, m.H / 8,
                      GatesEpi8T<true>{m, st, par}, s);
        if (part != 0)
            launch_s3(p.hBS, p.wpredS, p.nk_h, p.s3_per_h, p.s3_ks_h, p.s3_clu, m_tiles, p.proj_nt,
                      ProjEpi{m, st, par, h, set_cond}, s);
        return;
    }
    if (p.fk_lstm) {
        if (part != 1) {
            if (p.gates_ring)
                launch_gemm<128, GatesEpi>(p.hA, p.whh, m.H, 128, m_tiles, m.H / 32, GatesEpi{m, st, par}, s);
            else if (p.gates12)
                launch_fk<48, GatesEpi12>(p.hA3, p.whh3, p.nk_h, 48, m_tiles, (m.H + 11) / 12, GatesEpi12{m, st, par},
                                          s);
            else
                launch_fk<32, GatesEpi8>(p.hA3, p.whh3, p.nk_h, 32, m_tiles, m.H / 8, GatesEpi8{m, st, par}, s);
        }
        if (part != 0)
            launch_fk<32, ProjEpi>(p.hB3, p.wpred3, p.nk_h, 32, m_tiles, p.proj_nt, ProjEpi{m, st, par, h, set_cond},
                                   s);
        return;
    }
    if (part != 1) launch_gemm<128, GatesEpi>(p.hA, p.whh, m.H, 128, m_tiles, m.H / 32, GatesEpi{m, st, par}, s);
    if (part == 0) return;
    if (p.proj_mc)
        launch_gemm<32, ProjEpi, 4>(p.hB_mc, p.wpred, m.H, 32, m_tiles, p.proj_nt, ProjEpi{m, st, par, h, set_cond}, s);
    else
        launch_gemm<32, ProjEpi>(p.hB, p.wpred, m.H, 32, m_tiles, p.proj_nt, ProjEpi{m, st, par, h, set_cond}, s);
}

}  // namespace tbeam_dev
