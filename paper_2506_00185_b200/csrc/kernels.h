// Launchers of the sm_100a kernels (host-callable, stream-ordered, capturable).
#pragma once

#include <cuda_runtime.h>

#include "engine.cuh"

namespace tbeam_dev {

// kernels_simt.cu
void launch_enc_proj_simt(const DevModel& m, const DevState& st, int rows, cudaStream_t s);
void launch_joint_simt(const DevModel& m, const DevLm& lm, const DevCfg& cfg, const DevState& st,
                       cudaStream_t s);
void launch_lstm_simt(const DevModel& m, const DevCfg& cfg, const DevState& st, cudaStream_t s);
int simt_tile_cols();

// kernels_search.cu
void launch_init(const DevModel& m, const DevLm& lm, const DevCfg& cfg, const DevState& st,
                 cudaStream_t s);
void launch_select(const DevModel& m, const DevLm& lm, const DevCfg& cfg, const DevState& st,
                   cudaStream_t s);
void launch_pred_update(const DevModel& m, const DevCfg& cfg, const DevState& st, cudaStream_t s);
void launch_control(const DevState& st, cudaGraphConditionalHandle h, int use_handle,
                    cudaStream_t s);
void launch_finalize(const DevModel& m, const DevLm& lm, const DevCfg& cfg, const DevState& st,
                     cudaStream_t s);
size_t select_smem_bytes(int K, int ND);
void configure_kernels();

}  // namespace tbeam_dev
