// C-ABI of the B200 decoder (include/tbeam_b200.h): context, weight and LM
// upload, plan preparation (device buffers + the CUDA graph of the whole
// decode), decode entry points and result download.
//
// The graph of one decode (§2.1 "CUDA Graphs"; north star item 5):
//
//   enc_proj -> init -> WHILE(any stream unfinished) {
//                          2 x [ joint -> select (+ prediction-state gather)
//                                [-> LSTM gate GEMM -> projection GEMM] ]
//                          (the last select CTA sets the WHILE condition on device)
//                       } -> finalize
//
// so a decode is one cudaGraphLaunch with no host synchronisation inside.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/tbeam_b200.h"
#include "engine.cuh"
#include "kernels.h"
#include "lm_build.h"

using namespace tbeam_dev;

namespace {

thread_local std::string g_err;

struct CudaError {
    cudaError_t e;
    std::string where;
};

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t _e = (call);                                                          \
        if (_e != cudaSuccess) throw CudaError{_e, std::string(#call) + " @" + __FILE__ + \
                                                       ":" + std::to_string(__LINE__)};   \
    } while (0)

struct Status {
    int code;
    std::string msg;
};

// device buffer arena (freed together)
struct Arena {
    std::vector<void*> ptrs;
    template <class T>
    T* alloc(size_t n) {
        void* p = nullptr;
        if (n == 0) n = 1;
        CK(cudaMalloc(&p, n * sizeof(T)));
        CK(cudaMemset(p, 0, n * sizeof(T)));
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    template <class T>
    T* upload(const T* src, size_t n) {
        T* d = alloc<T>(n);
        if (src != nullptr && n > 0) CK(cudaMemcpy(d, src, n * sizeof(T), cudaMemcpyHostToDevice));
        return d;
    }
    void release() {
        for (void* p : ptrs) cudaFree(p);
        ptrs.clear();
    }
    ~Arena() { release(); }
};

double sigmoid(double x) { return 1.0 / (1.0 + std::exp(-x)); }

float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

struct PlanKey {
    tbeam_decode_config cfg;
    int B, Tmax;
    // semantic fields only: padding and reserved[] never force a re-capture
    bool operator==(const PlanKey& o) const {
        const tbeam_decode_config& a = cfg;
        const tbeam_decode_config& b = o.cfg;
        return B == o.B && Tmax == o.Tmax && a.algo == b.algo && a.beam == b.beam &&
               a.max_symbols_per_frame == b.max_symbols_per_frame &&
               a.aes_expansions_per_frame == b.aes_expansions_per_frame && a.max_len == b.max_len &&
               a.return_nbest == b.return_nbest && a.aes_prefix_search == b.aes_prefix_search &&
               a.lm_weight == b.lm_weight && a.blank_mode == b.blank_mode && a.prune_mode == b.prune_mode &&
               a.eos_enabled == b.eos_enabled && a.merge_mode == b.merge_mode && a.hash_base == b.hash_base &&
               a.hash_modulus == b.hash_modulus && a.aes_slot_donated_quirk == b.aes_slot_donated_quirk;
    }
};

}  // namespace

struct tbeam_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int graph_mode = 1;
    // model
    bool has_model = false;
    tbeam_model_dims dims{};
    DevModel dm{};
    Arena model_mem;
    // LM
    bool has_lm = false;
    tbeam_host::HostLm hlm;
    DevLm dl{};
    Arena lm_mem;
    // plan
    bool has_plan = false;
    PlanKey key{};
    DevCfg dc{};
    DevState ds{};
    Arena plan_mem;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t body_graph = nullptr;       // host-loop mode
    cudaGraphExec_t body_exec = nullptr;
    // input staging + indirection slots
    float* enc_buf = nullptr;
    size_t enc_cap = 0;
    int* len_buf = nullptr;
    int len_cap = 0;
    const float** d_enc_pp = nullptr;
    const int** d_len_pp = nullptr;
    // pipelined host-buffer decodes (tbeam_stage_inputs / tbeam_decode_staged):
    // two device input slots filled on a copy stream, FIFO of staged batches
    float* in_slot[2] = {nullptr, nullptr};
    int* len_slot[2] = {nullptr, nullptr};
    size_t in_cap[2] = {0, 0};
    int len_slot_cap[2] = {0, 0};
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t copied[2] = {nullptr, nullptr};
    int staged_batch[2] = {0, 0}, staged_frames[2] = {0, 0};
    int stage_head = 0, stage_count = 0;
    int per_round_kernels = 0;
    long long last_rounds = 0;
    TcPlan tc{};
    __nv_bfloat16* w_hh16_perm = nullptr;  // LSTM W_hh rows regrouped per 32 units x (i,f,g,o)
    // full-K GEMM operands: K padded (zeros) to a multiple of 64
    __nv_bfloat16* w_out16p = nullptr;     // [R+ND][Jk]
    __nv_bfloat16* w_pred16p = nullptr;    // [J][Hk]
    __nv_bfloat16* w_hh16g8 = nullptr;     // [4H][Hk], rows regrouped per 8 units x (i,f,g,o)
    __nv_bfloat16* w_hh16g12 = nullptr;    // [48 ceil(H/12)][Hk], rows regrouped per 12 units x (i,f,g,o)
    // precision fp32 on the tensor cores: the same padded layouts as three bf16
    // planes [3][rows][Kk] (device_fns.cuh put_op), NULL for a bf16 model
    __nv_bfloat16* w_out16s = nullptr;     // [3][R+ND][Jk]
    __nv_bfloat16* w_pred16s = nullptr;    // [3][J][Hk]
    __nv_bfloat16* w_hh16g8s = nullptr;    // [3][4H][Hk], 8-unit gate tiles

    void drop_plan() {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        if (body_exec) cudaGraphExecDestroy(body_exec);
        if (body_graph) cudaGraphDestroy(body_graph);
        exec = nullptr;
        graph = nullptr;
        body_exec = nullptr;
        body_graph = nullptr;
        plan_mem.release();
        has_plan = false;
    }
    ~tbeam_ctx() {
        drop_plan();
        model_mem.release();
        lm_mem.release();
        if (enc_buf) cudaFree(enc_buf);
        if (len_buf) cudaFree(len_buf);
        if (d_enc_pp) cudaFree(d_enc_pp);
        if (d_len_pp) cudaFree(d_len_pp);
        for (int k = 0; k < 2; ++k) {
            if (in_slot[k]) cudaFree(in_slot[k]);
            if (len_slot[k]) cudaFree(len_slot[k]);
            if (copied[k]) cudaEventDestroy(copied[k]);
        }
        if (copy_stream) cudaStreamDestroy(copy_stream);
        if (stream) cudaStreamDestroy(stream);
    }
};

namespace {

template <class F>
tbeam_status guarded(F&& f) {
    try {
        g_err.clear();
        Status s = f();
        if (s.code != TBEAM_OK) g_err = s.msg;
        return static_cast<tbeam_status>(s.code);
    } catch (const CudaError& e) {
        g_err = std::string("CUDA error ") + cudaGetErrorString(e.e) + " in " + e.where;
        return TBEAM_CUDA;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return TBEAM_CAPACITY;
    } catch (const std::exception& e) {
        g_err = e.what();
        return TBEAM_INVALID_ARGUMENT;
    }
}

// DecodeConfig validation: validate_streams (decoder.cpp:16-38)
Status validate_cfg(const tbeam_ctx* ctx, const tbeam_decode_config& c) {
    if (c.algo < 0 || c.algo > 2) return {TBEAM_INVALID_ARGUMENT, "decode: bad config (algo)"};
    if (c.beam < 1 || c.max_symbols_per_frame < 1 || c.aes_expansions_per_frame < 0 || c.max_len < 1 ||
        c.return_nbest < 1)
        return {TBEAM_INVALID_ARGUMENT, "decode: bad config"};
    if (c.lm_weight < 0.0) return {TBEAM_INVALID_ARGUMENT, "decode: negative LM weight"};
    if (c.lm_weight > 0.0 && !ctx->has_lm)
        return {TBEAM_INVALID_ARGUMENT, "decode: LM weight set but no LM given"};
    if (c.hash_modulus < 1) return {TBEAM_INVALID_ARGUMENT, "decode: hash modulus must be >= 1"};
    const int K = c.algo == TBEAM_ALGO_GREEDY ? 1 : c.beam;
    if (K > kMaxBeam)
        return {TBEAM_UNSUPPORTED, "decode: beam > " + std::to_string(kMaxBeam) + " not supported"};
    return {TBEAM_OK, ""};
}

void launch_joint(tbeam_ctx* ctx, int par, cudaStream_t s) {
    if (ctx->tc.enabled) launch_joint_tc(ctx->dm, ctx->dl, ctx->dc, ctx->ds, ctx->tc, par, s);
    else launch_joint_simt(ctx->dm, ctx->dl, ctx->dc, ctx->ds, par, s);
}

// LSTM token rows: gate GEMM + projection GEMM (the stateless network and the
// blank/dead children are updated inside the select kernel)
void launch_pred(tbeam_ctx* ctx, int par, cudaStream_t s, cudaGraphConditionalHandle h = {}, int set_cond = 0,
                 int part = -1) {
    if (ctx->dm.pred_kind != TBEAM_PRED_LSTM) return;
    if (ctx->tc.enabled) launch_lstm_tc(ctx->dm, ctx->ds, ctx->tc, par, h, set_cond, s, part);
    else launch_lstm_simt(ctx->dm, ctx->dc, ctx->ds, par, s, part);
}

// one round of the search for parity `par`; the round's last kernel sets the
// WHILE condition (the projection GEMM for a tensor-core LSTM, else select)
void launch_round(tbeam_ctx* ctx, int par, cudaGraphConditionalHandle h, int set_cond, cudaStream_t s) {
    launch_joint(ctx, par, s);
    const int in_proj = ctx->ds.round_in_proj;
    launch_select(ctx->dm, ctx->dl, ctx->dc, ctx->ds, par, h, in_proj ? 0 : set_cond, s);
    launch_pred(ctx, par, s, h, in_proj ? set_cond : 0);
}

void launch_prologue_encproj(tbeam_ctx* ctx, cudaStream_t s) {
    const int rows = ctx->ds.B * ctx->ds.Tmax;
    if (ctx->tc.enabled && !ctx->tc.s3) {  // (fp32: the CUDA-core projection, once per decode)
        launch_enc_to_bf16(ctx->dm, ctx->ds, rows, s);
        launch_encproj_tc(ctx->dm, ctx->ds, ctx->tc, rows, s);
    } else {
        launch_enc_proj_simt(ctx->dm, ctx->ds, rows, s);
    }
}

// WHILE body = two rounds (parity 0 then 1); the second select sets the loop
// condition.  A stream finishing after the first round makes the second a no-op.
// The body holds `pairs` round pairs (default 8): each WHILE iteration costs a
// graph relaunch, so unrolling amortises it; the few no-op rounds after the
// last stream finishes exit immediately (no rows) and are not counted.
void capture_body(tbeam_ctx* ctx, cudaStream_t s, cudaGraphConditionalHandle h, int use_handle) {
    int pairs = 8;
    if (const char* e = std::getenv("TBEAM_BODY_PAIRS")) pairs = std::max(1, std::min(16, std::atoi(e)));
    for (int q = 0; q < pairs; ++q) {
        launch_round(ctx, 0, h, 0, s);
        launch_round(ctx, 1, h, q == pairs - 1 ? use_handle : 0, s);
    }
}

// measurement aids compiled into the next captured plan (kernel parameters,
// so production plans pay nothing): 1 = phase trace, 2 = launch timeline
int g_trace_flags = 0;

// debug aid (tbeam_debug_round_trace): per-round slot state of one stream,
// recorded by the host loop (graph mode 0) after every round
int g_rt_stream = -1;
std::vector<double> g_rt_buf;

void record_round(tbeam_ctx* ctx, cudaStream_t s) {
    const DevState& st = ctx->ds;
    const int b = g_rt_stream, K = st.K;
    if (b < 0 || b >= st.B) return;
    std::vector<double> sc(K);
    std::vector<int> f(K), len(K), last(K);
    std::vector<unsigned long long> hs(K);
    int t = 0, r = 0, done = 0;
    CK(cudaMemcpyAsync(hs.data(), st.hash + static_cast<size_t>(b) * K, K * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(sc.data(), st.score + static_cast<size_t>(b) * K, K * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(f.data(), st.f + static_cast<size_t>(b) * K, K * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(len.data(), st.len + static_cast<size_t>(b) * K, K * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(last.data(), st.last + static_cast<size_t>(b) * K, K * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&t, st.t + b, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&r, st.r + b, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&done, st.done + b, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    g_rt_buf.push_back(t);
    g_rt_buf.push_back(r);
    g_rt_buf.push_back(done);
    g_rt_buf.push_back(0.0);  // (the oracle's record carries its prune margin here)
    g_rt_buf.push_back(0.0);
    for (int k = 0; k < K; ++k) {
        g_rt_buf.push_back(sc[k]);
        g_rt_buf.push_back(f[k]);
        g_rt_buf.push_back(len[k]);
        g_rt_buf.push_back(last[k]);
        g_rt_buf.push_back(static_cast<double>(hs[k] >> 32));
        g_rt_buf.push_back(static_cast<double>(hs[k] & 0xffffffffull));
    }
}

Status build_plan(tbeam_ctx* ctx, const tbeam_decode_config& c, int B, int Tmax) {
    ctx->drop_plan();
    const DevModel& m = ctx->dm;
    DevCfg dc{};
    dc.algo = c.algo;
    dc.K = c.algo == TBEAM_ALGO_GREEDY ? 1 : c.beam;
    dc.rounds = c.algo == TBEAM_ALGO_AES ? c.aes_expansions_per_frame + 1 : c.max_symbols_per_frame;
    dc.token_rounds = dc.rounds - 1;
    dc.max_len = c.max_len;
    dc.nbest = c.algo == TBEAM_ALGO_GREEDY ? 1 : c.return_nbest;
    dc.prefix = c.aes_prefix_search;
    dc.blank_mode = c.blank_mode;
    dc.prune_mode = c.prune_mode;
    dc.eos = c.eos_enabled;
    dc.merge_mode = c.merge_mode;
    dc.quirk = c.aes_slot_donated_quirk;
    dc.with_lm = ctx->has_lm && c.lm_weight > 0.0;
    dc.late = dc.with_lm && c.prune_mode == TBEAM_PRUNE_LATE;
    dc.early = dc.with_lm && c.prune_mode == TBEAM_PRUNE_EARLY;
    dc.lam = c.lm_weight;
    dc.hbase = c.hash_base;
    dc.hmod = c.hash_modulus;

    const int K = dc.K;
    const int S = B * K;
    const int ncols = m.R + m.ND;
    DevState st{};
    st.B = B;
    st.S = S;
    st.K = K;
    st.Tmax = Tmax;
    const bool lstm = m.pred_kind == TBEAM_PRED_LSTM;
    const char* force_simt = std::getenv("TBEAM_FORCE_SIMT");
    TcPlan tp{};
    tp.enabled = m.prec == TBEAM_PREC_BF16 && m.J % 8 == 0 && m.D % 8 == 0 &&
                 (!lstm || (m.H % 32 == 0 && ctx->w_hh16_perm != nullptr)) &&
                 !(force_simt && force_simt[0] == '1');
    // precision fp32: the tensor-core GEMMs on three-plane operands (tc_gemm_s3,
    // BN = 32 tiles, k-block accumulators summed in fp64) unless
    // TBEAM_FP32_SIMT=1 keeps the CUDA-core FFMA kernels (measurement switch)
    const char* fp32_simt = std::getenv("TBEAM_FP32_SIMT");
    const int nt32 = (ncols + 31) / 32;
    tp.s3 = m.prec == TBEAM_PREC_FP32 && ctx->w_out16s != nullptr && m.J % 8 == 0 &&
            (!lstm || (m.H % 8 == 0 && ctx->w_hh16g8s != nullptr && ctx->w_pred16s != nullptr)) && nt32 <= 256 &&
            1LL * nt32 * K <= 2048 && !(force_simt && force_simt[0] == '1') && !(fp32_simt && fp32_simt[0] == '1');
    if (tp.s3) {
        // k-blocks per CTA (<= 3: one 3-D box per plane) and K slices per tile
        auto slices = [](int nk, int& per, int& ks) {
            ks = (nk + 2) / 3;
            per = (nk + ks - 1) / ks;
            if (const char* e = std::getenv("TBEAM_S3_PER")) {  // test / measurement override
                const int v = std::atoi(e);
                if (v >= 1 && v <= 3) per = std::min(v, nk);
            }
            ks = (nk + per - 1) / per;
        };
        tp.nk_j = (m.J + 63) / 64;
        tp.nk_h = (std::max(m.H, 1) + 63) / 64;
        slices(tp.nk_j, tp.s3_per_j, tp.s3_ks_j);
        slices(tp.nk_h, tp.s3_per_h, tp.s3_ks_h);
        // K slices reduced through global memory + an arrival ticket (the last
        // slice to finish sums them).  TBEAM_S3_CLUSTER=1: the slices of a tile
        // as one cluster reduced through DSMEM -- measured slower (C2 40.0 ->
        // 41.6 ms per decode: slice 0 waits for the slowest slice at the
        // cluster barrier, and 4-CTA clusters of 204-KB CTAs leave SMs idle
        // per GPC: gates release skew 10 -> 15 us)
        const char* ce = std::getenv("TBEAM_S3_CLUSTER");
        tp.s3_clu = std::max(tp.s3_ks_j, tp.s3_ks_h) <= 8 && ce && ce[0] == '1';
        const long long m_tiles = (S + 127) / 128;
        const long long tiles = m_tiles * std::max<long long>({nt32, lstm ? m.H / 8 : 0, lstm ? (m.J + 31) / 32 : 0});
        const long long ksm = std::max(tp.s3_ks_j, lstm ? tp.s3_ks_h : 1);
        if (ksm > 1 && tiles * ksm * 4 * 128 * 8 * sizeof(double) > (512ll << 20)) tp.s3 = 0;  // partials too large
    }
    if (tp.s3) {
        tp.enabled = 1;
        tp.joint_bn = tp.joint_bnv = 32;
        tp.joint_nt = nt32;
        tp.joint_cl = 0;
        st.ntile_cols = 8;
        st.NT = nt32;
        tp.proj_nt = (m.J + 31) / 32;
    } else if (tp.enabled) {
        tp.joint_bn = S <= 2048 ? 32 : S <= 8192 ? 64 : 256;
        // late LM fusion makes the epilogue the joint's long pole: from 1024
        // rows on, 64-column tiles keep the grid in one wave (measured C4:
        // 33.6 -> 27.5 us per joint launch)
        if (dc.late && S >= 1024 && tp.joint_bn == 32) tp.joint_bn = 64;
        // one wave: the full-K BN = 32 joint runs one 208-KB CTA per SM, so
        // past one wave of (M-tile, N-tile) CTAs the 64-column ring tiles win
        // (measured C3, S = 1024: 264 CTAs -> 136; ALSD++ 186.5K -> 202.7K RTFx,
        // AES++ 173.5K -> 182.6K; the bench's 132 CTAs stay at BN = 32)
        {
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
            const long long cta32 = 1LL * ((S + 127) / 128) * ((ncols + 31) / 32);
            if (tp.joint_bn == 32 && cta32 > sms) tp.joint_bn = 64;
        }
        if (const char* e = std::getenv("TBEAM_JOINT_BN")) {  // measurement override
            const int v = std::atoi(e);
            if (v == 32 || v == 64 || v == 256) tp.joint_bn = v;
        }
        // the select kernel merges NT x K partial candidates per row (one
        // list per joint tile; the epilogue merges its 4 sub-blocks in smem):
        // <= 256 lists, <= 2048 entries
        auto parts = [&](int bn) { return 1LL * ((ncols + bn - 1) / bn); };
        while (tp.joint_bn < 256 && (parts(tp.joint_bn) * K > 2048 || parts(tp.joint_bn) > 256))
            tp.joint_bn = tp.joint_bn == 32 ? 64 : 256;
        int nt = (ncols + tp.joint_bn - 1) / tp.joint_bn;
        tp.joint_bnv = std::min(tp.joint_bn, ((ncols + nt - 1) / nt + 31) / 32 * 32);
        // 4-CTA multicast of z when every k-block has its own stage; the grid's
        // N extent is padded to the cluster (padded tiles emit empty partials)
        // opt-in (TBEAM_MULTICAST=1): measured no faster at the bench shape,
        // where the mainloop is latency- not L2-bandwidth-bound
        const char* mc_env = std::getenv("TBEAM_MULTICAST");
        const bool mc_ok = mc_env && mc_env[0] == '1';
        tp.joint_mc = 0;  // the joint reads z once per tile column group; no multicast variant
        tp.joint_nt = nt;
        st.ntile_cols = tp.joint_bnv / 4;
        st.NT = nt;
        // ring joints (BN 64 / 256) at K 5..16 with many tile columns: clusters
        // of CL CTAs along N can merge their per-row lists through DSMEM, so
        // the select stages NT / CL lists per row instead of NT (C5: 33 -> 5);
        // the N grid is padded to a multiple of CL (padded tiles emit empty
        // lists).  Opt-in (TBEAM_JOINT_CLUSTER = auto / 4 / 8): measured slower
        // -- C4 46.5 -> 65.8 ms, C5 1492 -> 1984 ms per decode: the per-row
        // 8-way merge (K warp-wide picks over DSMEM) and the padded, cluster-
        // scheduled grid cost more than the partial traffic saves.
        tp.joint_cl = 0;
        const bool ring = tp.joint_bn >= 64 && K >= 5 && K <= 16;
        const char* cl_env = std::getenv("TBEAM_JOINT_CLUSTER");
        if (ring && nt >= 8 && cl_env && std::strcmp(cl_env, "auto") == 0) {
            for (int cl : {8, 4}) {
                const int padded = (nt + cl - 1) / cl * cl;
                if (4 * (padded - nt) <= nt) {
                    tp.joint_cl = cl;
                    break;
                }
            }
        }
        if (cl_env && std::strcmp(cl_env, "auto") != 0) {
            const int v = std::atoi(cl_env);
            tp.joint_cl = (ring && (v == 4 || v == 8)) ? v : 0;
        }
        if (tp.joint_cl > 1) {
            tp.joint_nt = (nt + tp.joint_cl - 1) / tp.joint_cl * tp.joint_cl;
            st.NT = tp.joint_nt / tp.joint_cl;
        }
        tp.proj_nt = (m.J + 31) / 32;
        tp.proj_mc = mc_ok && lstm && (m.H + 63) / 64 <= tc_stages_for(32);
        if (tp.proj_mc) tp.proj_nt = (tp.proj_nt + 3) / 4 * 4;
    } else {
        st.ntile_cols = simt_tile_cols(ncols, K);
        st.NT = (ncols + st.ntile_cols - 1) / st.ntile_cols;
    }
    // split-K for the CUDA-core GEMMs while the tiles alone cannot fill the GPU
    // (decode row counts): 8 or 4 slices of the K loop per tile (TBEAM_SPLITK
    // overrides: 1 / 2 / 4 / 8)
    st.sk_split = 1;
    if (tp.s3) {
        const long long m_tiles = (S + 127) / 128;
        const long long tiles = m_tiles * std::max<long long>({st.NT, lstm ? m.H / 8 : 0, lstm ? tp.proj_nt : 0});
        const long long ksm = std::max(tp.s3_ks_j, lstm ? tp.s3_ks_h : 1);
        if (ksm > 1) {
            st.sk_scratch = ctx->plan_mem.alloc<double>(static_cast<size_t>(tiles * ksm) * 4 * 128 * 8);
            st.sk_ticket = ctx->plan_mem.alloc<unsigned>(static_cast<size_t>(tiles));
            CK(cudaMemset(st.sk_ticket, 0, static_cast<size_t>(tiles) * sizeof(unsigned)));
        }
    } else if (!tp.enabled) {
        const long long row_tiles = (S + 31) / 32;
        const long long tiles = std::max<long long>({row_tiles * st.NT, lstm ? row_tiles * ((m.H + 7) / 8) : 0,
                                                    lstm ? row_tiles * ((m.J + 31) / 32) : 0});
        st.sk_split = row_tiles <= 4 ? 8 : row_tiles <= 8 ? 4 : 1;  // (C2: 1 / 2 / 4 / 8 slices:
                                                                  //  121 / 100 / 85 / 81 us per round)
        if (const char* e = std::getenv("TBEAM_SPLITK")) {
            const int v = std::atoi(e);
            if (v == 1 || v == 2 || v == 4 || v == 8) st.sk_split = v;
        }
        if (st.sk_split > 1) {
            const int cj = st.ntile_cols / 32 > 1 ? st.ntile_cols / 32 : 1;
            st.sk_scratch = ctx->plan_mem.alloc<double>(static_cast<size_t>(tiles) * st.sk_split * 256 * 4 * cj);
            st.sk_ticket = ctx->plan_mem.alloc<unsigned>(static_cast<size_t>(tiles));
            CK(cudaMemset(st.sk_ticket, 0, static_cast<size_t>(tiles) * sizeof(unsigned)));
        }
    }
    st.tc = tp.enabled;
    st.split3 = tp.s3;
    st.trace = g_trace_flags;
    st.round_in_proj = tp.enabled && lstm ? 1 : 0;
    st.probe_on = tp.enabled && dc.algo == TBEAM_ALGO_AES && dc.prefix && K <= 8 ? 1 : 0;
    st.Jp = (m.J + 63) / 64 * 64;  // K-padded (zeros): full-K 3-D TMA boxes read whole k-blocks
    st.Hp = (std::max(m.H, 1) + 63) / 64 * 64;
    st.Dp = (m.D + 7) / 8 * 8;
    st.ndx = m.ND > 0 ? m.ND : 1;
    if (static_cast<long long>(st.NT) * K > 2048 || st.NT > 256)
        return {TBEAM_UNSUPPORTED, "decode: (V+1)/tile * beam too large for the top-K merge"};
    st.max_cols = Tmax * dc.rounds + 1;
    Arena& a = ctx->plan_mem;
    st.T = a.alloc<int>(B);
    st.t = a.alloc<int>(B);
    st.r = a.alloc<int>(B);
    st.done = a.alloc<int>(B);
    st.steps = a.alloc<int>(B);
    st.ctr = a.alloc<unsigned long long>(static_cast<size_t>(B) * 5);
    st.score = a.alloc<double>(S);
    st.len = a.alloc<int>(S);
    st.hash = a.alloc<unsigned long long>(S);
    st.last = a.alloc<int>(S);
    st.f = a.alloc<int>(S);
    st.tnode = a.alloc<int>(S);
    st.lm_state = a.alloc<int>(S);
    st.donated = a.alloc<unsigned char>(S);
    st.sdonated = a.alloc<unsigned char>(S);
    st.P = 2 * K;
    const size_t prow = static_cast<size_t>(B) * st.P;
    st.pid = a.alloc<int>(S);
    st.win = a.alloc<int>(prow * std::max(m.n, 1));
    if (m.pred_kind == TBEAM_PRED_LSTM) {
        st.h = a.alloc<float>(prow * m.H);
        st.c = a.alloc<float>(prow * m.H);
    }
    st.pred = a.alloc<float>(prow * m.J);
    st.upd_src = a.alloc<int>(2ull * S);
    st.upd_dst = a.alloc<int>(2ull * S);
    st.upd_tok = a.alloc<int>(2ull * S);
    st.act_list = a.alloc<int>(2ull * S);
    st.act_count = a.alloc<int>(2);
    st.upd_list = a.alloc<int>(2ull * S);
    st.upd_count = a.alloc<int>(2);
    const size_t nt = static_cast<size_t>(S) * st.NT;
    st.part = a.alloc<float>(nt * part_stride(K));
    st.blank_logit = a.alloc<float>(S);
    st.dur_logit = a.alloc<float>(static_cast<size_t>(S) * st.ndx);
    const size_t cols = static_cast<size_t>(st.max_cols);
    st.st_tok = a.alloc<int>(cols * S);
    st.st_prev = a.alloc<int>(cols * S);
    st.st_dur = a.alloc<signed char>(cols * S);
    st.st_frame = a.alloc<int>(cols * B);
    st.encp = a.alloc<float>(static_cast<size_t>(B) * Tmax * m.J);
    st.enc_pp = ctx->d_enc_pp;
    st.len_pp = ctx->d_len_pp;
    st.g = a.alloc<int>(1);
    st.live = a.alloc<int>(1);
    st.probe = a.alloc<float>(static_cast<size_t>(S) * K);
    st.n_done = a.alloc<int>(1);
    st.sel_blocks = a.alloc<int>(1);
    st.col = a.alloc<int>(B);
    st.out_count = a.alloc<int>(B);
    st.out_len = a.alloc<int>(static_cast<size_t>(B) * dc.nbest);
    st.out_score = a.alloc<double>(static_cast<size_t>(B) * dc.nbest);
    const size_t ob = static_cast<size_t>(B) * dc.nbest * c.max_len;
    st.out_tok = a.alloc<int>(ob);
    st.out_frame = a.alloc<int>(ob);
    st.out_dur = a.alloc<int>(ob);
    st.zpl = static_cast<size_t>(S) * st.Jp;
    st.hpl = static_cast<size_t>(S) * st.Hp;
    if (tp.s3) {
        const int np = 3;
        st.z16 = a.alloc<__nv_bfloat16>(np * st.zpl);
        st.act_pos = a.alloc<int>(S);
        st.upd_pos = a.alloc<int>(S);
        const int rb[3] = {32, 64, 128};
        for (int q = 0; q < 3; ++q) tp.zS[q] = make_tc_map4(st.z16, S, tp.nk_j, st.Jp, st.zpl, rb[q], tp.s3_per_j);
        tp.woutS = make_tc_map4(ctx->w_out16s, ncols, tp.nk_j, tp.nk_j * 64, static_cast<size_t>(ncols) * tp.nk_j * 64,
                                32, tp.s3_per_j);
        if (lstm) {
            st.hA16 = a.alloc<__nv_bfloat16>(np * st.hpl);
            st.hB16 = a.alloc<__nv_bfloat16>(np * st.hpl);
            for (int q = 0; q < 3; ++q) {
                tp.hAS[q] = make_tc_map4(st.hA16, S, tp.nk_h, st.Hp, st.hpl, rb[q], tp.s3_per_h);
                tp.hBS[q] = make_tc_map4(st.hB16, S, tp.nk_h, st.Hp, st.hpl, rb[q], tp.s3_per_h);
            }
            const size_t hk = static_cast<size_t>(tp.nk_h) * 64;
            tp.whhS = make_tc_map4(ctx->w_hh16g8s, 4 * m.H, tp.nk_h, tp.nk_h * 64, 4 * m.H * hk, 32, tp.s3_per_h);
            tp.wpredS = make_tc_map4(ctx->w_pred16s, m.J, tp.nk_h, tp.nk_h * 64, m.J * hk, 32, tp.s3_per_h);
        }
    } else if (tp.enabled) {
        st.z16 = a.alloc<__nv_bfloat16>(static_cast<size_t>(S) * st.Jp);
        st.act_pos = a.alloc<int>(S);
        st.upd_pos = a.alloc<int>(S);
        st.enc16 = a.alloc<__nv_bfloat16>(static_cast<size_t>(B) * Tmax * st.Dp);
        tp.z = make_tc_map(st.z16, S, m.J, st.Jp, 32);  // A operands: 32-row boxes (live rows only)
        tp.z_mc = make_tc_map(st.z16, S, m.J, st.Jp, 32);
        tp.wout = make_tc_map(m.w_out16, ncols, m.J, m.J, tp.joint_bnv);
        tp.enc = make_tc_map(st.enc16, B * Tmax, m.D, st.Dp, 32);
        tp.wenc = make_tc_map(m.w_enc16, m.J, m.D, m.D, 128);
        if (lstm) {
            st.hA16 = a.alloc<__nv_bfloat16>(static_cast<size_t>(S) * st.Hp);
            st.hB16 = a.alloc<__nv_bfloat16>(static_cast<size_t>(S) * st.Hp);
            tp.hA = make_tc_map(st.hA16, S, m.H, st.Hp, 32);
            tp.whh = make_tc_map(ctx->w_hh16_perm, 4 * m.H, m.H, m.H, 128);
            tp.hB = make_tc_map(st.hB16, S, m.H, st.Hp, 32);
            tp.hB_mc = make_tc_map(st.hB16, S, m.H, st.Hp, 32);
            tp.wpred = make_tc_map(m.w_pred16, m.J, m.H, m.H, 32);
        }
        // full-K single-box GEMMs (K <= 640): joint at BN = 32, both LSTM GEMMs
        const bool no_fk = std::getenv("TBEAM_NO_FK") && std::getenv("TBEAM_NO_FK")[0] == '1';
        tp.nk_j = (m.J + 63) / 64;
        tp.nk_h = (std::max(m.H, 1) + 63) / 64;
        tp.fk_joint = !no_fk && tp.joint_bn == 32 && tp.nk_j <= 10 && ctx->w_out16p != nullptr;
        tp.fk_lstm = !no_fk && lstm && tp.nk_h <= 10 && m.H % 8 == 0 && ctx->w_hh16g8 != nullptr &&
                     ctx->w_pred16p != nullptr;
        const int rb[3] = {32, 64, 128};
        if (tp.fk_joint) {
            // A boxes of a fraction of the k-blocks (tc_gemm_fk loads A in several boxes)
            for (int q = 0; q < 3; ++q) tp.zA[q] = make_tc_map3(st.z16, S, tp.nk_j, st.Jp, rb[q], fk_abox_depth(tp.nk_j));
            tp.wout3 = make_tc_map3(ctx->w_out16p, ncols, tp.nk_j, tp.nk_j * 64, tp.joint_bnv);
        }
        if (tp.fk_lstm) {
            for (int q = 0; q < 3; ++q) {
                tp.hA3[q] = make_tc_map3(st.hA16, S, tp.nk_h, st.Hp, rb[q], fk_abox_depth(tp.nk_h));
                tp.hB3[q] = make_tc_map3(st.hB16, S, tp.nk_h, st.Hp, rb[q], fk_abox_depth(tp.nk_h));
            }
            // 12-unit gate tiles only with TBEAM_GATES12=1: measured slower at the
            // bench shape (gates 6.9 -> 11.2 us busy, DESIGN.md §8 rejected list)
            const char* g12env = std::getenv("TBEAM_GATES12");
            tp.gates12 = g12env && g12env[0] == '1' && ctx->w_hh16g12 != nullptr;
            // many token rows: the gates as the ring GEMM of 32-unit tiles --
            // 4x fewer CTAs than the 8-unit full-K tiles, whose M-tiles of
            // token rows then run in several waves.  Measured (same box,
            // TBEAM_GATES_RING=0 vs 1): C3 ALSD++ (B x K = 1024) 200.3K ->
            // 206.2K RTFx (gates 13.3 -> 11.4 us per round), C3 AES++ equal,
            // C4 AES++ 110.2K -> 108.4K, C5 (16,384 slots) 82.6K -> 89.4K; the
            // full-K projection stays (the ring one: C3 5.7 -> 9.6 us).
            // TBEAM_GATES_RING=0|1 overrides.
            tp.gates_ring = !tp.gates12 && m.H % 32 == 0 && ctx->w_hh16_perm != nullptr &&
                            (S >= 2048 || (S >= 1024 && dc.algo == TBEAM_ALGO_ALSD));
            if (const char* e = std::getenv("TBEAM_GATES_RING"))
                tp.gates_ring = (e[0] == '1') && m.H % 32 == 0 && ctx->w_hh16_perm != nullptr;
            if (tp.gates12)
                tp.whh3 = make_tc_map3(ctx->w_hh16g12, (m.H + 11) / 12 * 48, tp.nk_h, tp.nk_h * 64, 48);
            else
                tp.whh3 = make_tc_map3(ctx->w_hh16g8, 4 * m.H, tp.nk_h, tp.nk_h * 64, 32);
            tp.wpred3 = make_tc_map3(ctx->w_pred16p, m.J, tp.nk_h, tp.nk_h * 64, 32);
        }
    }
    ctx->tc = tp;
    ctx->dc = dc;
    ctx->ds = st;
    ctx->per_round_kernels = 2 + (m.pred_kind == TBEAM_PRED_LSTM ? 2 : 0);

    // ---- the decode graph -------------------------------------------------------
    cudaStream_t s = ctx->stream;
    if (ctx->graph_mode == 1) {
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        launch_prologue_encproj(ctx, s);
        launch_init(m, ctx->dl, dc, st, s);
        cudaStreamCaptureStatus cs;
        cudaGraph_t g = nullptr;
        const cudaGraphNode_t* deps = nullptr;
        size_t ndeps = 0;
        CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &ndeps));
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp{};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t cnode;
        CK(cudaGraphAddNode(&cnode, g, deps, ndeps, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        CK(cudaStreamUpdateCaptureDependencies(s, &cnode, 1, cudaStreamSetCaptureDependencies));
        launch_finalize(m, ctx->dl, dc, st, s);
        CK(cudaStreamEndCapture(s, &ctx->graph));
        cudaStream_t bs;
        CK(cudaStreamCreateWithFlags(&bs, cudaStreamNonBlocking));
        CK(cudaStreamBeginCaptureToGraph(bs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        capture_body(ctx, bs, h, 1);
        cudaGraph_t body_out = nullptr;
        CK(cudaStreamEndCapture(bs, &body_out));
        CK(cudaStreamDestroy(bs));
        CK(cudaGraphInstantiate(&ctx->exec, ctx->graph, 0));
    }
    ctx->key = PlanKey{c, B, Tmax};
    ctx->has_plan = true;
    return {TBEAM_OK, ""};
}

Status ensure_plan(tbeam_ctx* ctx, const tbeam_decode_config& c, int B, int Tmax) {
    if (!ctx->has_model) return {TBEAM_INVALID_ARGUMENT, "decode: no model set"};
    Status v = validate_cfg(ctx, c);
    if (v.code != TBEAM_OK) return v;
    if (B < 1) return {TBEAM_INVALID_ARGUMENT, "decode: no streams"};
    if (Tmax < 1) return {TBEAM_INVALID_ARGUMENT, "decode: bad stream input"};
    const PlanKey k{c, B, Tmax};
    if (ctx->has_plan && ctx->key == k && ctx->ds.trace == g_trace_flags) return {TBEAM_OK, ""};
    return build_plan(ctx, c, B, Tmax);
}

void run_plan(tbeam_ctx* ctx, cudaStream_t s) {
    if (ctx->graph_mode == 1) {
        CK(cudaGraphLaunch(ctx->exec, s));
        return;
    }
    const DevModel& m = ctx->dm;
    launch_prologue_encproj(ctx, s);
    launch_init(m, ctx->dl, ctx->dc, ctx->ds, s);
    int n_done = 0;
    for (long long it = 0; it < ctx->ds.max_cols;) {
        // plain stream launches (profilers cannot instrument graph nodes that
        // may set a conditional handle)
        for (int q = 0; q < 8 && it < ctx->ds.max_cols; ++q, it += 2) {
            launch_round(ctx, 0, cudaGraphConditionalHandle{}, 0, s);
            if (g_rt_stream >= 0) record_round(ctx, s);
            launch_round(ctx, 1, cudaGraphConditionalHandle{}, 0, s);
            if (g_rt_stream >= 0) record_round(ctx, s);
        }
        CK(cudaMemcpyAsync(&n_done, ctx->ds.n_done, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (n_done >= ctx->ds.B) break;
    }
    launch_finalize(m, ctx->dl, ctx->dc, ctx->ds, s);
}

void set_inputs(tbeam_ctx* ctx, const float* enc_dev, const int* len_dev, cudaStream_t s) {
    static_assert(sizeof(const float*) == 8, "64-bit");
    CK(cudaMemcpyAsync(ctx->d_enc_pp, &enc_dev, sizeof(enc_dev), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(ctx->d_len_pp, &len_dev, sizeof(len_dev), cudaMemcpyHostToDevice, s));
}

Status fetch(tbeam_ctx* ctx, tbeam_results* res, cudaStream_t s) {
    const DevState& st = ctx->ds;
    const int B = st.B, nb = ctx->dc.nbest, L = ctx->key.cfg.max_len;
    if (res == nullptr) return {TBEAM_OK, ""};
    if (res->batch != B || res->nbest < nb || res->max_len < L)
        return {TBEAM_INVALID_ARGUMENT, "results: buffer shape does not match the decode"};
    std::vector<int> cnt(B), len(static_cast<size_t>(B) * nb);
    std::vector<double> sc(static_cast<size_t>(B) * nb);
    const size_t ob = static_cast<size_t>(B) * nb * L;
    std::vector<int> tok(ob), fr(ob), du(ob);
    std::vector<unsigned long long> ctr(static_cast<size_t>(B) * 5);
    CK(cudaMemcpyAsync(cnt.data(), st.out_count, B * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(len.data(), st.out_len, len.size() * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(sc.data(), st.out_score, sc.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(tok.data(), st.out_tok, ob * sizeof(int), cudaMemcpyDeviceToHost, s));
    if (res->frames) CK(cudaMemcpyAsync(fr.data(), st.out_frame, ob * sizeof(int), cudaMemcpyDeviceToHost, s));
    if (res->durations) CK(cudaMemcpyAsync(du.data(), st.out_dur, ob * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ctr.data(), st.ctr, ctr.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    int g = 0;
    CK(cudaMemcpyAsync(&g, st.g, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    ctx->last_rounds = g;
    for (int b = 0; b < B; ++b) {
        res->nbest_count[b] = cnt[b];
        for (int r = 0; r < res->nbest; ++r) {
            const size_t e = static_cast<size_t>(b) * res->nbest + r;
            const size_t se = static_cast<size_t>(b) * nb + r;
            res->lengths[e] = r < nb ? len[se] : 0;
            res->scores[e] = r < nb ? sc[se] : -INFINITY;
            if (r >= nb) continue;
            for (int u = 0; u < len[se] && u < res->max_len; ++u) {
                res->tokens[e * res->max_len + u] = tok[se * L + u];
                if (res->frames) res->frames[e * res->max_len + u] = fr[se * L + u];
                if (res->durations) res->durations[e * res->max_len + u] = du[se * L + u];
            }
        }
        if (res->counters)
            for (int q = 0; q < 5; ++q) res->counters[static_cast<size_t>(b) * 5 + q] = ctr[static_cast<size_t>(b) * 5 + q];
    }
    return {TBEAM_OK, ""};
}

}  // namespace

extern "C" {

void tbeam_decode_config_init(tbeam_decode_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->algo = TBEAM_ALGO_ALSD;
    c->beam = 4;
    c->max_symbols_per_frame = 10;
    c->aes_expansions_per_frame = 2;
    c->max_len = 256;
    c->return_nbest = 1;
    c->aes_prefix_search = 1;
    c->lm_weight = 0.0;
    c->blank_mode = TBEAM_BLANK_OMIT;
    c->prune_mode = TBEAM_PRUNE_LATE;
    c->eos_enabled = 0;
    c->merge_mode = TBEAM_MERGE_LOGSUMEXP;
    c->hash_base = 1000003ull;
    c->hash_modulus = (1ull << 61) - 1;
    c->aes_slot_donated_quirk = 0;
}

const char* tbeam_last_error(void) { return g_err.c_str(); }
int32_t tbeam_abi_version(void) { return TBEAM_B200_ABI_VERSION; }

tbeam_status tbeam_create(int device, tbeam_ctx** out) {
    return guarded([&]() -> Status {
        if (out == nullptr) return {TBEAM_INVALID_ARGUMENT, "create: null out"};
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
            return {TBEAM_UNSUPPORTED, "create: no CUDA device"};
        if (device < 0 || device >= n) return {TBEAM_INVALID_ARGUMENT, "create: bad device index"};
        cudaDeviceProp prop{};
        CK(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10 || prop.minor != 0)
            return {TBEAM_UNSUPPORTED, "create: kernels are built for sm_100a (B200); device is sm_" +
                                           std::to_string(prop.major) + std::to_string(prop.minor)};
        CK(cudaSetDevice(device));
        auto ctx = std::make_unique<tbeam_ctx>();
        ctx->device = device;
        // TBEAM_GRAPH_MODE=0: start in host-loop mode (sanitizers / profilers
        // that do not follow conditional graph nodes)
        if (const char* e = std::getenv("TBEAM_GRAPH_MODE")) ctx->graph_mode = e[0] == '0' ? 0 : 1;
        CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        CK(cudaMalloc(&ctx->d_enc_pp, sizeof(void*)));
        CK(cudaMalloc(&ctx->d_len_pp, sizeof(void*)));
        configure_kernels();
        configure_tc_kernels();
        *out = ctx.release();
        return {TBEAM_OK, ""};
    });
}

tbeam_status tbeam_destroy(tbeam_ctx* ctx) {
    if (ctx) {
        cudaSetDevice(ctx->device);
        delete ctx;
    }
    return TBEAM_OK;
}

tbeam_status tbeam_set_graph_mode(tbeam_ctx* ctx, int32_t mode) {
    return guarded([&]() -> Status {
        if (!ctx || (mode != 0 && mode != 1)) return {TBEAM_INVALID_ARGUMENT, "graph mode must be 0 or 1"};
        CK(cudaSetDevice(ctx->device));
        if (ctx->graph_mode != mode) {
            ctx->graph_mode = mode;
            ctx->drop_plan();
        }
        return {TBEAM_OK, ""};
    });
}

tbeam_status tbeam_set_model(tbeam_ctx* ctx, const tbeam_model_dims* d, const tbeam_model_weights* w) {
    return guarded([&]() -> Status {
        if (!ctx || !d || !w) return {TBEAM_INVALID_ARGUMENT, "set_model: null argument"};
        CK(cudaSetDevice(ctx->device));
        const int V = d->vocab_size, D = d->enc_dim, J = d->joint_dim, ND = d->num_durations;
        const bool lstm = d->pred_kind == TBEAM_PRED_LSTM;
        const int H = lstm ? d->lstm_hidden : 0, E = lstm ? d->emb_dim : 0;
        if (V < 1 || D < 1 || J < 1 || ND < 0 || ND > TBEAM_MAX_DURATIONS || d->pred_kind < 0 ||
            d->pred_kind > 1 || (!lstm && (d->context_order < 0 || d->context_order > 64)) ||
            (lstm && (H < 1 || E < 1 || H % 4 != 0 || J % 4 != 0)) || d->precision < 0 || d->precision > 1)
            return {TBEAM_INVALID_ARGUMENT, "set_model: bad dimensions"};
        for (int i = 0; i < ND; ++i)
            if (d->durations[i] < 0 || (i > 0 && d->durations[i] <= d->durations[i - 1]))
                return {TBEAM_INVALID_ARGUMENT, "set_model: durations must be ascending and >= 0"};
        if (ND > 0 && d->durations[ND - 1] < 1)
            return {TBEAM_INVALID_ARGUMENT, "set_model: TDT needs a duration >= 1"};
        if (!w->w_enc || !w->b_enc || !w->b_pred || !w->w_out || !w->b_out || (ND > 0 && (!w->w_dur || !w->b_dur)) ||
            (!lstm && !w->pred_table) || (lstm && (!w->emb || !w->w_ih || !w->w_hh || !w->b_lstm || !w->w_pred)))
            return {TBEAM_INVALID_ARGUMENT, "set_model: missing weight"};
        if (ctx->has_lm && d->vocab_size != ctx->dl.V)
            return {TBEAM_VALIDATION, "set_model: vocabulary size differs from the loaded LM's"};
        ctx->drop_plan();
        // invalidate before freeing: an upload that throws below leaves no
        // model behind instead of dangling device pointers
        ctx->has_model = false;
        ctx->dm = DevModel{};
        ctx->model_mem.release();
        ctx->w_hh16_perm = nullptr;
        ctx->w_out16p = ctx->w_pred16p = ctx->w_hh16g8 = ctx->w_hh16g12 = nullptr;
        ctx->w_out16s = ctx->w_pred16s = ctx->w_hh16g8s = nullptr;
        Arena& a = ctx->model_mem;
        const int R = V + 1;
        const bool bf = d->precision == TBEAM_PREC_BF16;
        DevModel m{};
        m.V = V;
        m.R = R;
        m.D = D;
        m.J = J;
        m.H = H;
        m.E = E;
        m.ND = ND;
        m.n = lstm ? 0 : d->context_order;
        m.pred_kind = d->pred_kind;
        m.prec = d->precision;
        m.di0 = -1;
        for (int i = 0; i < ND; ++i) {
            m.durations[i] = d->durations[i];
            if (d->durations[i] == 0) m.di0 = i;
        }
        auto to_bf16 = [&](const float* src, size_t n) {
            std::vector<__nv_bfloat16> v(n);
            for (size_t i = 0; i < n; ++i) v[i] = __float2bfloat16_rn(src[i]);
            return a.upload(v.data(), n);
        };
        m.w_enc = a.upload(w->w_enc, static_cast<size_t>(J) * D);
        m.b_enc = a.upload(w->b_enc, J);
        m.b_pred = a.upload(w->b_pred, J);
        // output projection: token rows then duration rows
        const size_t nrows = static_cast<size_t>(R) + ND;
        std::vector<float> wo(nrows * J), bo(nrows);
        std::memcpy(wo.data(), w->w_out, sizeof(float) * R * J);
        std::memcpy(bo.data(), w->b_out, sizeof(float) * R);
        if (ND > 0) {
            std::memcpy(wo.data() + static_cast<size_t>(R) * J, w->w_dur, sizeof(float) * ND * J);
            std::memcpy(bo.data() + R, w->b_dur, sizeof(float) * ND);
        }
        m.w_out = a.upload(wo.data(), wo.size());
        m.b_out = a.upload(bo.data(), bo.size());
        // K-padded bf16 copy: [rows][kp], zeros beyond k
        auto to_bf16_pad = [&](const float* src, size_t rows, int k, int kp) {
            std::vector<__nv_bfloat16> v(rows * kp, __float2bfloat16_rn(0.f));
            for (size_t r = 0; r < rows; ++r)
                for (int c = 0; c < k; ++c) v[r * kp + c] = __float2bfloat16_rn(src[r * k + c]);
            return a.upload(v.data(), v.size());
        };
        // the three-plane split of the same layout (fp32 models)
        auto to_bf16_pad3 = [&](const float* src, size_t rows, int k, int kp) {
            std::vector<__nv_bfloat16> v(3 * rows * kp, __float2bfloat16_rn(0.f));
            for (size_t r = 0; r < rows; ++r)
                for (int c = 0; c < k; ++c) {
                    float x = src[r * k + c];
                    for (int p = 0; p < 3; ++p) {
                        const __nv_bfloat16 h = __float2bfloat16_rn(x);
                        v[(p * rows + r) * kp + c] = h;
                        x -= __bfloat162float(h);
                    }
                }
            return a.upload(v.data(), v.size());
        };
        const int Jk = (J + 63) / 64 * 64, Hk = (H + 63) / 64 * 64;
        if (bf) {
            m.w_enc16 = to_bf16(w->w_enc, static_cast<size_t>(J) * D);
            m.w_out16 = to_bf16(wo.data(), wo.size());
            ctx->w_out16p = to_bf16_pad(wo.data(), nrows, J, Jk);
        } else {
            ctx->w_out16s = to_bf16_pad3(wo.data(), nrows, J, Jk);
        }
        if (lstm) {
            // input half of every LSTM step as a table: X[v] = W_ih . emb[v] + b
            std::vector<double> xt(static_cast<size_t>(R) * 4 * H);
            for (int v = 0; v < R; ++v)
                for (int q = 0; q < 4 * H; ++q) {
                    double acc = 0.0;
                    const float* wr = w->w_ih + static_cast<size_t>(q) * E;
                    const float* er = w->emb + static_cast<size_t>(v) * E;
                    for (int e = 0; e < E; ++e) acc += static_cast<double>(wr[e]) * er[e];
                    xt[static_cast<size_t>(v) * 4 * H + q] = acc + w->b_lstm[q];
                }
            std::vector<float> xf(xt.begin(), xt.end());
            m.xtab = a.upload(xf.data(), xf.size());
            m.w_hh = a.upload(w->w_hh, 4ull * H * H);
            m.w_pred = a.upload(w->w_pred, static_cast<size_t>(J) * H);
            if (!bf) {
                ctx->w_pred16s = to_bf16_pad3(w->w_pred, J, H, Hk);
                if (H % 8 == 0) {  // 8-unit gate tiles, as the bf16 full-K layout below
                    std::vector<float> g8(4ull * H * H);
                    for (int nt = 0; nt < H / 8; ++nt)
                        for (int gate = 0; gate < 4; ++gate)
                            for (int u = 0; u < 8; ++u)
                                std::memcpy(g8.data() + (static_cast<size_t>(nt) * 32 + gate * 8 + u) * H,
                                            w->w_hh + (static_cast<size_t>(gate) * H + nt * 8 + u) * H,
                                            sizeof(float) * H);
                    ctx->w_hh16g8s = to_bf16_pad3(g8.data(), 4ull * H, H, Hk);
                }
            }
            if (bf) {
                m.w_hh16 = to_bf16(w->w_hh, 4ull * H * H);
                m.w_pred16 = to_bf16(w->w_pred, static_cast<size_t>(J) * H);
                if (H % 32 == 0) {
                    // tensor-core gate tile nt = units [32nt, 32nt+32) x gates (i,f,g,o):
                    // permuted row nt*128 + gate*32 + u  <-  W_hh row gate*H + 32nt + u
                    std::vector<float> perm(4ull * H * H);
                    for (int nt = 0; nt < H / 32; ++nt)
                        for (int gate = 0; gate < 4; ++gate)
                            for (int u = 0; u < 32; ++u)
                                std::memcpy(perm.data() + (static_cast<size_t>(nt) * 128 + gate * 32 + u) * H,
                                            w->w_hh + (static_cast<size_t>(gate) * H + nt * 32 + u) * H,
                                            sizeof(float) * H);
                    ctx->w_hh16_perm = to_bf16(perm.data(), perm.size());
                }
                ctx->w_pred16p = to_bf16_pad(w->w_pred, J, H, Hk);
                if (H % 8 == 0) {
                    // full-K gate tile nt = units [8nt, 8nt+8) x gates (i,f,g,o):
                    // row nt*32 + gate*8 + u  <-  W_hh row gate*H + 8nt + u
                    std::vector<float> g8(4ull * H * H);
                    for (int nt = 0; nt < H / 8; ++nt)
                        for (int gate = 0; gate < 4; ++gate)
                            for (int u = 0; u < 8; ++u)
                                std::memcpy(g8.data() + (static_cast<size_t>(nt) * 32 + gate * 8 + u) * H,
                                            w->w_hh + (static_cast<size_t>(gate) * H + nt * 8 + u) * H,
                                            sizeof(float) * H);
                    ctx->w_hh16g8 = to_bf16_pad(g8.data(), 4ull * H, H, Hk);
                }
                {
                    // 12-unit gate tile nt: row nt*48 + gate*12 + u  <-  W_hh row
                    // gate*H + 12nt + u (zero rows past H)
                    const int nt12 = (H + 11) / 12;
                    std::vector<float> g12(static_cast<size_t>(nt12) * 48 * H, 0.f);
                    for (int nt = 0; nt < nt12; ++nt)
                        for (int gate = 0; gate < 4; ++gate)
                            for (int u = 0; u < 12 && nt * 12 + u < H; ++u)
                                std::memcpy(g12.data() + (static_cast<size_t>(nt) * 48 + gate * 12 + u) * H,
                                            w->w_hh + (static_cast<size_t>(gate) * H + nt * 12 + u) * H,
                                            sizeof(float) * H);
                    ctx->w_hh16g12 = to_bf16_pad(g12.data(), static_cast<size_t>(nt12) * 48, H, Hk);
                }
            }
            // start state: one step from zeros with the BOS row (X[V])
            std::vector<float> h0(H), c0(H), p0(J);
            const double* x = xt.data() + static_cast<size_t>(V) * 4 * H;
            for (int u = 0; u < H; ++u) {
                const double ig = sigmoid(x[u]), gg = std::tanh(x[2 * H + u]), og = sigmoid(x[3 * H + u]);
                const double cn = ig * gg;
                c0[u] = static_cast<float>(cn);
                h0[u] = static_cast<float>(og * std::tanh(cn));
            }
            for (int j = 0; j < J; ++j) {
                double acc = 0.0;
                for (int u = 0; u < H; ++u) {
                    const float hv = bf ? bf16r(h0[u]) : h0[u];
                    const float wv = bf ? bf16r(w->w_pred[static_cast<size_t>(j) * H + u])
                                        : w->w_pred[static_cast<size_t>(j) * H + u];
                    acc += static_cast<double>(wv) * hv;
                }
                p0[j] = static_cast<float>(acc + w->b_pred[j]);
            }
            m.h0 = a.upload(h0.data(), H);
            m.c0 = a.upload(c0.data(), H);
            m.pred0 = a.upload(p0.data(), J);
        } else {
            m.table = a.upload(w->pred_table, static_cast<size_t>(R) * J);
        }
        ctx->dm = m;
        ctx->dims = *d;
        ctx->has_model = true;
        return {TBEAM_OK, ""};
    });
}

tbeam_status tbeam_set_lm_arpa(tbeam_ctx* ctx, const char* text, size_t len, const char* const* tokens,
                               int32_t vocab_size, int32_t strict) {
    return guarded([&]() -> Status {
        if (!ctx || !text || !tokens || vocab_size < 1) return {TBEAM_INVALID_ARGUMENT, "set_lm: bad argument"};
        if (ctx->has_model && vocab_size != ctx->dm.V)
            return {TBEAM_VALIDATION, "set_lm: vocabulary size differs from the model's"};
        CK(cudaSetDevice(ctx->device));
        std::vector<std::string> vocab(tokens, tokens + vocab_size);
        tbeam_host::HostLm h;
        std::string err;
        const int rc = tbeam_host::build_lm(text, len, vocab, strict != 0, h, err);
        if (rc != 0) return {rc, err};
        if (h.order > kMaxOrder + 1)
            return {TBEAM_UNSUPPORTED, "set_lm: n-gram order " + std::to_string(h.order) + " > " +
                                           std::to_string(kMaxOrder + 1) + " (device backoff chain limit)"};
        ctx->drop_plan();
        ctx->has_lm = false;
        ctx->dl = DevLm{};
        ctx->lm_mem.release();
        Arena& a = ctx->lm_mem;
        DevLm d{};
        d.present = 1;
        d.order = h.order;
        d.V = h.V;
        d.initial = h.initial;
        d.prob = a.upload(h.prob.data(), h.prob.size());
        d.backoff = a.upload(h.backoff.data(), h.backoff.size());
        d.suffix = a.upload(h.suffix.data(), h.suffix.size());
        d.depth = a.upload(h.depth.data(), h.depth.size());
        d.cbeg = a.upload(h.cbeg.data(), h.cbeg.size());
        d.cend = a.upload(h.cend.data(), h.cend.size());
        d.etok = a.upload(h.etok.data(), h.etok.size());
        d.enode = a.upload(h.enode.data(), h.enode.size());
        d.remap = a.upload(h.remap.data(), h.remap.size());
        d.uni = a.upload(h.uni.data(), h.uni.size());
        d.root = a.upload(h.root.data(), h.root.size());
        d.n_root = static_cast<int>(h.root.size());
        d.unk_prob = h.unk_prob;
        ctx->hlm = std::move(h);
        ctx->dl = d;
        ctx->has_lm = true;
        return {TBEAM_OK, ""};
    });
}

tbeam_status tbeam_lm_parse_check(const char* text, size_t len, const char* const* tokens, int32_t vocab_size,
                                  int32_t strict, int64_t out[4]) {
    return guarded([&]() -> Status {
        if (!text || !tokens || vocab_size < 1 || !out) return {TBEAM_INVALID_ARGUMENT, "parse_check: bad argument"};
        std::vector<std::string> vocab(tokens, tokens + vocab_size);
        tbeam_host::HostLm h;
        std::string err;
        const int rc = tbeam_host::build_lm(text, len, vocab, strict != 0, h, err);
        if (rc != 0) return {rc, err};
        if (h.order > kMaxOrder + 1)
            return {TBEAM_UNSUPPORTED, "set_lm: n-gram order " + std::to_string(h.order) + " > " +
                                           std::to_string(kMaxOrder + 1) + " (device backoff chain limit)"};
        out[0] = h.order;
        out[1] = static_cast<int64_t>(h.prob.size());
        out[2] = static_cast<int64_t>(h.etok.size());
        out[3] = static_cast<int64_t>(h.oov_mapped);
        return {TBEAM_OK, ""};
    });
}

tbeam_status tbeam_clear_lm(tbeam_ctx* ctx) {
    return guarded([&]() -> Status {
        if (!ctx) return {TBEAM_INVALID_ARGUMENT, "null ctx"};
        ctx->drop_plan();
        ctx->lm_mem.release();
        ctx->dl = DevLm{};
        ctx->has_lm = false;
        return {TBEAM_OK, ""};
    });
}

tbeam_status tbeam_lm_export(const char* text, size_t len, const char* const* tokens, int32_t vocab_size,
                             int32_t strict, int64_t out[4], double* prob, double* backoff, int32_t* suffix,
                             int32_t* depth, int32_t* cbeg, int32_t* cend, int32_t* etok, int32_t* enode,
                             int32_t* remap) {
    return guarded([&]() -> Status {
        if (!text || !tokens || vocab_size < 1 || !out) return {TBEAM_INVALID_ARGUMENT, "lm_export: bad argument"};
        std::vector<std::string> vocab(tokens, tokens + vocab_size);
        tbeam_host::HostLm h;
        std::string err;
        const int rc = tbeam_host::build_lm(text, len, vocab, strict != 0, h, err);
        if (rc != 0) return {rc, err};
        out[0] = h.order;
        out[1] = static_cast<int64_t>(h.prob.size());
        out[2] = static_cast<int64_t>(h.etok.size());
        out[3] = h.initial;
        auto put = [](auto* dst, const auto& v) {
            if (dst) std::copy(v.begin(), v.end(), dst);
        };
        put(prob, h.prob);
        put(backoff, h.backoff);
        put(suffix, h.suffix);
        put(depth, h.depth);
        put(cbeg, h.cbeg);
        put(cend, h.cend);
        put(etok, h.etok);
        put(enode, h.enode);
        put(remap, h.remap);
        return {TBEAM_OK, ""};
    });
}

tbeam_status tbeam_lm_info(tbeam_ctx* ctx, int64_t out[4]) {
    if (!ctx || !out) return TBEAM_INVALID_ARGUMENT;
    out[0] = ctx->has_lm ? ctx->hlm.order : 0;
    out[1] = ctx->has_lm ? static_cast<int64_t>(ctx->hlm.prob.size()) : 0;
    out[2] = ctx->has_lm ? static_cast<int64_t>(ctx->hlm.etok.size()) : 0;
    out[3] = ctx->has_lm ? static_cast<int64_t>(ctx->hlm.oov_mapped) : 0;
    return TBEAM_OK;
}

tbeam_status tbeam_prepare(tbeam_ctx* ctx, const tbeam_decode_config* cfg, int32_t batch, int32_t max_frames) {
    return guarded([&]() -> Status {
        if (!ctx || !cfg) return {TBEAM_INVALID_ARGUMENT, "prepare: null argument"};
        CK(cudaSetDevice(ctx->device));
        return ensure_plan(ctx, *cfg, batch, max_frames);
    });
}

tbeam_status tbeam_decode_device(tbeam_ctx* ctx, const float* enc_dev, const int32_t* lengths_dev, void* stream) {
    return guarded([&]() -> Status {
        if (!ctx || !ctx->has_plan) return {TBEAM_INVALID_ARGUMENT, "decode_device: call tbeam_prepare first"};
        if (!enc_dev || !lengths_dev) return {TBEAM_INVALID_ARGUMENT, "decode_device: null input"};
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
        set_inputs(ctx, enc_dev, lengths_dev, s);
        run_plan(ctx, s);
        return {TBEAM_OK, ""};
    });
}

tbeam_status tbeam_fetch_results(tbeam_ctx* ctx, tbeam_results* res, void* stream) {
    return guarded([&]() -> Status {
        if (!ctx || !ctx->has_plan) return {TBEAM_INVALID_ARGUMENT, "fetch: nothing decoded"};
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
        return fetch(ctx, res, s);
    });
}

tbeam_status tbeam_decode(tbeam_ctx* ctx, const tbeam_decode_config* cfg, const float* enc, int32_t on_device,
                          const int32_t* lengths, int32_t batch, int32_t max_frames, tbeam_results* res,
                          void* stream) {
    return guarded([&]() -> Status {
        if (!ctx || !cfg || !enc || !lengths) return {TBEAM_INVALID_ARGUMENT, "decode: null argument"};
        CK(cudaSetDevice(ctx->device));
        if (batch < 1) return {TBEAM_INVALID_ARGUMENT, "decode: no streams"};
        for (int b = 0; b < batch; ++b)
            if (lengths[b] < 1 || lengths[b] > max_frames) return {TBEAM_INVALID_ARGUMENT, "decode: bad stream input"};
        Status st = ensure_plan(ctx, *cfg, batch, max_frames);
        if (st.code != TBEAM_OK) return st;
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
        const size_t n = static_cast<size_t>(batch) * max_frames * ctx->dm.D;
        const float* enc_dev = enc;
        if (!on_device) {
            if (ctx->enc_cap < n) {
                if (ctx->enc_buf) CK(cudaFree(ctx->enc_buf));
                CK(cudaMalloc(&ctx->enc_buf, n * sizeof(float)));
                ctx->enc_cap = n;
            }
            CK(cudaMemcpyAsync(ctx->enc_buf, enc, n * sizeof(float), cudaMemcpyHostToDevice, s));
            enc_dev = ctx->enc_buf;
        }
        if (ctx->len_cap < batch) {
            if (ctx->len_buf) CK(cudaFree(ctx->len_buf));
            CK(cudaMalloc(&ctx->len_buf, batch * sizeof(int)));
            ctx->len_cap = batch;
        }
        CK(cudaMemcpyAsync(ctx->len_buf, lengths, batch * sizeof(int), cudaMemcpyHostToDevice, s));
        set_inputs(ctx, enc_dev, ctx->len_buf, s);
        run_plan(ctx, s);
        return fetch(ctx, res, s);
    });
}

tbeam_status tbeam_stage_inputs(tbeam_ctx* ctx, const float* enc_host, const int32_t* lengths, int32_t batch,
                                int32_t max_frames) {
    return guarded([&]() -> Status {
        if (!ctx || !enc_host || !lengths) return {TBEAM_INVALID_ARGUMENT, "stage: null argument"};
        if (!ctx->has_model) return {TBEAM_INVALID_ARGUMENT, "decode: no model set"};
        if (batch < 1) return {TBEAM_INVALID_ARGUMENT, "decode: no streams"};
        if (max_frames < 1) return {TBEAM_INVALID_ARGUMENT, "decode: bad stream input"};
        for (int b = 0; b < batch; ++b)
            if (lengths[b] < 1 || lengths[b] > max_frames) return {TBEAM_INVALID_ARGUMENT, "decode: bad stream input"};
        if (ctx->stage_count >= 2) return {TBEAM_INVALID_ARGUMENT, "stage: two batches already staged"};
        CK(cudaSetDevice(ctx->device));
        if (!ctx->copy_stream) {
            CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
            for (int k = 0; k < 2; ++k) CK(cudaEventCreateWithFlags(&ctx->copied[k], cudaEventDisableTiming));
        }
        const int k = (ctx->stage_head + ctx->stage_count) & 1;
        const size_t n = static_cast<size_t>(batch) * max_frames * ctx->dm.D;
        if (ctx->in_cap[k] < n) {
            if (ctx->in_slot[k]) CK(cudaFree(ctx->in_slot[k]));
            CK(cudaMalloc(&ctx->in_slot[k], n * sizeof(float)));
            ctx->in_cap[k] = n;
        }
        if (ctx->len_slot_cap[k] < batch) {
            if (ctx->len_slot[k]) CK(cudaFree(ctx->len_slot[k]));
            CK(cudaMalloc(&ctx->len_slot[k], batch * sizeof(int)));
            ctx->len_slot_cap[k] = batch;
        }
        CK(cudaMemcpyAsync(ctx->in_slot[k], enc_host, n * sizeof(float), cudaMemcpyHostToDevice, ctx->copy_stream));
        CK(cudaMemcpyAsync(ctx->len_slot[k], lengths, batch * sizeof(int), cudaMemcpyHostToDevice, ctx->copy_stream));
        CK(cudaEventRecord(ctx->copied[k], ctx->copy_stream));
        ctx->staged_batch[k] = batch;
        ctx->staged_frames[k] = max_frames;
        ++ctx->stage_count;
        return {TBEAM_OK, ""};
    });
}

tbeam_status tbeam_decode_staged(tbeam_ctx* ctx, const tbeam_decode_config* cfg, tbeam_results* res, void* stream) {
    return guarded([&]() -> Status {
        if (!ctx || !cfg) return {TBEAM_INVALID_ARGUMENT, "decode: null argument"};
        if (ctx->stage_count < 1) return {TBEAM_INVALID_ARGUMENT, "decode: nothing staged"};
        CK(cudaSetDevice(ctx->device));
        const int k = ctx->stage_head;
        const int batch = ctx->staged_batch[k], max_frames = ctx->staged_frames[k];
        // the batch leaves the queue whatever happens below (the call is
        // synchronous: slot k is free again when it returns)
        ctx->stage_head ^= 1;
        --ctx->stage_count;
        Status st = ensure_plan(ctx, *cfg, batch, max_frames);
        if (st.code != TBEAM_OK) return st;
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
        CK(cudaStreamWaitEvent(s, ctx->copied[k], 0));
        set_inputs(ctx, ctx->in_slot[k], ctx->len_slot[k], s);
        run_plan(ctx, s);
        return fetch(ctx, res, s);  // synchronises s
    });
}

int32_t tbeam_profile_decode(tbeam_ctx* ctx, const float* enc_dev, const int32_t* lengths_dev, void* stream,
                             double* ms_out, int64_t* launches_out, int64_t* rows_out) {
    int32_t families = -1;
    const tbeam_status st = guarded([&]() -> Status {
        if (!ctx || !ctx->has_plan || !enc_dev || !lengths_dev || !ms_out || !launches_out || !rows_out)
            return {TBEAM_INVALID_ARGUMENT, "profile: prepare first / null argument"};
        CK(cudaSetDevice(ctx->device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
        constexpr int NF = 7;
        for (int f = 0; f < NF; ++f) {
            ms_out[f] = 0.0;
            launches_out[f] = 0;
        }
        std::vector<cudaEvent_t> ev;
        std::vector<int> fam;  // family of the interval ending at event i
        auto mark = [&](int f) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            CK(cudaEventRecord(e, s));
            ev.push_back(e);
            fam.push_back(f);
        };
        const DevModel& m = ctx->dm;
        set_inputs(ctx, enc_dev, lengths_dev, s);
        mark(-1);
        launch_prologue_encproj(ctx, s);
        mark(0);
        launch_init(m, ctx->dl, ctx->dc, ctx->ds, s);
        mark(1);
        int n_done = 0;
        long long rounds = 0;
        while (rounds < ctx->ds.max_cols) {
            for (int q = 0; q < 16 && rounds < ctx->ds.max_cols; ++q, ++rounds) {
                const int par = static_cast<int>(rounds & 1);
                launch_joint(ctx, par, s);
                mark(2);
                launch_select(m, ctx->dl, ctx->dc, ctx->ds, par, cudaGraphConditionalHandle{}, 0, s);
                mark(3);
                if (m.pred_kind == TBEAM_PRED_LSTM) {
                    launch_pred(ctx, par, s, {}, 0, 0);
                    mark(4);
                    launch_pred(ctx, par, s, {}, 0, 1);
                    mark(5);
                }
            }
            CK(cudaMemcpyAsync(&n_done, ctx->ds.n_done, sizeof(int), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (n_done >= ctx->ds.B) break;
        }
        launch_finalize(m, ctx->dl, ctx->dc, ctx->ds, s);
        mark(6);
        CK(cudaStreamSynchronize(s));
        for (size_t i = 1; i < ev.size(); ++i) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, ev[i - 1], ev[i]));
            ms_out[fam[i]] += ms;
            launches_out[fam[i]] += 1;
        }
        // rounds actually executed until every stream finished
        int g = 0;
        CK(cudaMemcpy(&g, ctx->ds.g, sizeof(int), cudaMemcpyDeviceToHost));
        std::vector<unsigned long long> ctr(static_cast<size_t>(ctx->ds.B) * 5);
        CK(cudaMemcpy(ctr.data(), ctx->ds.ctr, ctr.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        long long scored = 0;
        for (int b = 0; b < ctx->ds.B; ++b) scored += static_cast<long long>(ctr[b * 5 + 2]);
        rows_out[0] = scored;
        rows_out[1] = g;
        for (cudaEvent_t e : ev) cudaEventDestroy(e);
        families = NF;
        return {TBEAM_OK, ""};
    });
    return st == TBEAM_OK ? families : -1;
}

// measurement aid (not in the public header): accumulate the phase trace of
// tc_gemm CTA (0,0) -- out = {launches, prologue, dependency wait, mainloop,
// epilogue} in SM cycles -- and reset it; enable = 1 to keep tracing.
// out = 40 GEMM slots, then [1024 select CTAs][8] phase accumulators.
int32_t tbeam_debug_gemm_trace(int32_t enable, int64_t* out) {
    g_trace_flags = enable ? (g_trace_flags | 1) : (g_trace_flags & ~1);  // next prepare re-captures
    long long o[40];
    std::vector<long long> q(1024 * 32);
    gemm_trace(enable, o);
    sel_trace(enable, q.data());
    if (out) {
        for (int i = 0; i < 40; ++i) out[i] = o[i];
        for (int i = 0; i < 1024 * 32; ++i) out[40 + i] = q[i];  // select phases per CTA
    }
    return 0;
}

// measurement aid: device-wide launch timeline, out = [4096 rounds][4 kernels
// (joint, gates, proj, select)][4 stamps (first entry, first release, last
// release, last exit)] in globaltimer ns (0 / ~0 = no launch); resets it.
int32_t tbeam_debug_timeline(int32_t enable, uint64_t* out) {
    g_trace_flags = enable ? (g_trace_flags | 2) : (g_trace_flags & ~2);  // next prepare re-captures
    std::vector<unsigned long long> a(4096 * 16), b(4096 * 16);
    tl_read_tc(enable, out ? a.data() : nullptr);
    tl_read_sel(enable, out ? b.data() : nullptr);
    if (out)
        for (size_t r = 0; r < 4096; ++r)
            for (int k = 0; k < 4; ++k)
                for (int q = 0; q < 4; ++q) out[(r * 4 + k) * 4 + q] = k == 3 ? b[(r * 4 + k) * 4 + q] : a[(r * 4 + k) * 4 + q];
    return 0;
}

// debug aid: stream >= 0 starts recording stream `stream`'s per-round slot
// state in host-loop decodes (set_graph_mode(0)); stream < 0 stops.  Returns
// the number of doubles recorded so far and copies up to `cap` of them to out
// (record = t, r, done, 0, 0, then per slot: score, f, len, last, hash >> 32,
// hash & 0xffffffff); with out != null
// the record is copied and cleared.
int64_t tbeam_debug_round_trace(int32_t stream, double* out, int64_t cap) {
    const int64_t n = static_cast<int64_t>(g_rt_buf.size());
    if (out)
        for (int64_t i = 0; i < n && i < cap; ++i) out[i] = g_rt_buf[static_cast<size_t>(i)];
    if (out) g_rt_buf.clear();
    g_rt_stream = stream;
    return n;
}

int32_t tbeam_launch_stats(tbeam_ctx* ctx, int64_t* out, int32_t cap) {
    if (!ctx || !out || cap < 1) return 0;
    // prologue (enc_proj, init) + rounds x per-round kernels + finalize
    const int64_t total = 3 + ctx->last_rounds * ctx->per_round_kernels;
    out[0] = total;
    if (cap > 1) out[1] = ctx->last_rounds;
    if (cap > 2) out[2] = ctx->per_round_kernels;
    return cap > 2 ? 3 : cap;
}

}  // extern "C"
