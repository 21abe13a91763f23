// Launchers of the sm_100a kernels (host-callable, stream-ordered, capturable).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "engine.cuh"

namespace tbeam_dev {

// kernels_tc.cu (tcgen05 / TMEM / TMA)
struct TcMap {
    CUtensorMap map;
};
struct TcPlan {
    int enabled = 0;
    int fk_joint = 0, fk_lstm = 0, nk_j = 0, nk_h = 0;  // full-K single-box GEMMs (tc_gemm_fk)
    int gates12 = 0;  // LSTM gates in 12-unit (N = 48) tiles (else 8-unit, N = 32)
    int gates_ring = 0;  // LSTM gates as the ring GEMM (128-column tiles: 32 units x 4 gates) beside the full-K projection
    TcMap zA[3], wout3, hA3[3], whh3, hB3[3], wpred3;    // 3-D maps: A boxes of 32/64/128 rows
    int joint_bn = 64, joint_bnv = 64, joint_nt = 1;  // joint_nt: N extent of the grid (padded to joint_cl)
    int joint_cl = 0;  // > 1: clusters of joint_cl CTAs along N merge their tile lists (JointEpi<.., CLU>)
    int joint_mc = 0, proj_mc = 0, proj_nt = 1;  // 4-CTA cluster multicast of the A operand
    TcMap z, wout, enc, wenc, hA, whh, hB, wpred, z_mc, hB_mc;
    // precision fp32 on the tensor cores (tc_gemm_s3): operands as three bf16
    // planes stacked along the rows; per = k-blocks per CTA (<= 3), ks = K slices
    int s3 = 0, s3_per_j = 1, s3_ks_j = 1, s3_per_h = 1, s3_ks_h = 1;
    int s3_clu = 0;  // 1: the K slices of a tile run as one cluster, reduced through DSMEM (opt-in)
    TcMap zS[3], woutS, hAS[3], hBS[3], whhS, wpredS;  // 4-D plane maps, box depth = per
};
TcMap make_tc_map(const void* base, int rows, int k, int pitch_elems, int box_rows);
// 3-D map {64, rows, nk} (k-block stride 128 B); a box is {64, box_rows,
// depth} (depth 0 = nk: every k-block of the tile)
TcMap make_tc_map3(const void* base, int rows, int nk, int pitch_elems, int box_rows, int depth = 0);
// 4-D map over three stacked bf16 planes {64, rows, 3, nk} (plane stride
// plane_elems): a box {64, box_rows, 3, depth} lands as [k-block][plane][rows]
TcMap make_tc_map4(const void* base, int rows, int nk, int pitch_elems, size_t plane_elems, int box_rows, int depth);
void configure_tc_kernels();
int fk_abox_depth(int nk);  // k-blocks per A box of the full-K GEMMs
void gemm_trace(int enable, long long* out);
int tc_stages_for(int bn);
void launch_joint_tc(const DevModel& m, const DevLm& lm, const DevCfg& cfg, const DevState& st, const TcPlan& p,
                     int par, cudaStream_t s);
void launch_encproj_tc(const DevModel& m, const DevState& st, const TcPlan& p, int rows, cudaStream_t s);
// part: -1 both GEMMs, 0 the gates only, 1 the projection only (profiling)
void launch_lstm_tc(const DevModel& m, const DevState& st, const TcPlan& p, int par, cudaGraphConditionalHandle h,
                    int set_cond, cudaStream_t s, int part = -1);
void launch_enc_to_bf16(const DevModel& m, const DevState& st, int rows, cudaStream_t s);

// kernels_simt.cu
void launch_enc_proj_simt(const DevModel& m, const DevState& st, int rows, cudaStream_t s);
void launch_joint_simt(const DevModel& m, const DevLm& lm, const DevCfg& cfg, const DevState& st, int par,
                       cudaStream_t s);
void launch_lstm_simt(const DevModel& m, const DevCfg& cfg, const DevState& st, int par, cudaStream_t s,
                      int part = -1);
int simt_tile_cols(int ncols, int K);

// kernels_search.cu
void launch_init(const DevModel& m, const DevLm& lm, const DevCfg& cfg, const DevState& st,
                 cudaStream_t s);
void launch_select(const DevModel& m, const DevLm& lm, const DevCfg& cfg, const DevState& st, int par,
                   cudaGraphConditionalHandle h, int set_cond, cudaStream_t s);
void launch_finalize(const DevModel& m, const DevLm& lm, const DevCfg& cfg, const DevState& st,
                     cudaStream_t s);
size_t select_smem_bytes(int K, int ND, int NT);
int select_threads(int K);
void configure_kernels();
void sel_trace(int enable, long long* out);
// launch timeline tables [kTlRounds][4 kernels][4 stamps] (tc_common.cuh); read + reset
void tl_read_tc(int enable, unsigned long long* out);
void tl_read_sel(int enable, unsigned long long* out);

}  // namespace tbeam_dev
