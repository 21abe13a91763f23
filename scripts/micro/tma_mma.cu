// TMA + tcgen05 pipeline microbenchmark (measurement aid): how long do nk
// k-blocks of a 128 x BN x 64 tile take to land in smem and be consumed by
// UMMA, as a function of bytes, grid size and MMA presence?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_2506_00185_b200/csrc -o tma_mma tma_mma.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <vector>
#include "tc_common.cuh"
using namespace tbeam_dev;

constexpr int BK = 64, BM = 128;

template <int BN, int NK>
__global__ void __launch_bounds__(128, 1) pipe(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                                               int do_mma, int arows, unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    constexpr int AB = BM * BK * 2, BB = BN * BK * 2;
    uint8_t* sA = smem;
    uint8_t* sB = smem + NK * AB;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + NK * BB);
    uint64_t* done = full + NK;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
    if (threadIdx.x == 0) {
        for (int s = 0; s < NK; ++s) mbar_init(&full[s], 1);
        mbar_init(done, 1);
        mbar_fence_init();
    }
    if (threadIdx.x < 32) tmem_alloc(tslot, BN < 32 ? 32 : BN);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const long long t0 = clock64();
    long long tarr[NK];
    if (threadIdx.x == 0) {
        const int nbox = (arows + 31) / 32;
        for (int kb = 0; kb < NK; ++kb) {
            mbar_expect_tx(&full[kb], nbox * 32 * BK * 2 + BB);
            for (int i = 0; i < nbox; ++i) tma_load_2d(sA + kb * AB + i * 32 * BK * 2, &ta, &full[kb], kb * BK, 32 * i);
            tma_load_2d(sB + kb * BB, &tb, &full[kb], kb * BK, 0);
        }
    } else if (threadIdx.x == 32) {
        const uint32_t idesc = umma_idesc_bf16(BM, BN);
        for (int kb = 0; kb < NK; ++kb) {
            mbar_wait(&full[kb], 0);
            tarr[kb] = clock64() - t0;
            tc_fence_after();
            if (do_mma) {
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                    umma_bf16(tmem, umma_desc_sw128(smem_u32(sA + kb * AB) + 32 * k),
                              umma_desc_sw128(smem_u32(sB + kb * BB) + 32 * k), idesc, (kb | k) ? 1u : 0u);
            }
        }
        if (do_mma) umma_commit(done);
        else mbar_expect_tx(done, 0);
        mbar_wait(done, 0);
        const long long t1 = clock64() - t0;
        if (blockIdx.x == 0) {
            for (int kb = 0; kb < NK; ++kb) out[kb] = tarr[kb];
            out[NK] = t1;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem, BN < 32 ? 32 : BN);
}

PFN_cuTensorMapEncodeTiled_v12000 enc_fn;
CUtensorMap mk(void* p, int rows, int k, int box_rows) {
    CUtensorMap t;
    cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)rows};
    cuuint64_t str[1] = {(cuuint64_t)k * 2};
    cuuint32_t box[2] = {BK, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    enc_fn(&t, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return t;
}

template <int BN, int NK>
void run(const char* name, int grid, int do_mma, int arows, void* A, void* Bm, unsigned long long* out) {
    CUtensorMap ta = mk(A, 128, NK * BK, 32), tb = mk(Bm, BN, NK * BK, BN);
    const int smem = 1024 + NK * (BM * BK * 2 + BN * BK * 2) + 256;
    cudaFuncSetAttribute(pipe<BN, NK>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 3; ++rep) pipe<BN, NK><<<grid, 128, smem>>>(ta, tb, do_mma, arows, out);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<unsigned long long> h(NK + 1);
    cudaMemcpy(h.data(), out, 8 * (NK + 1), cudaMemcpyDeviceToHost);
    printf("%-34s grid=%3d mma=%d arows=%3d: arrivals", name, grid, do_mma, arows);
    for (int i = 0; i < NK; ++i) printf(" %llu", h[i]);
    printf(" | done %llu  (%s)\n", h[NK], cudaGetErrorString(e));
}

int main() {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc_fn), cudaEnableDefault, &q);
    void *A, *B;
    unsigned long long* out;
    cudaMalloc(&A, 128 * 640 * 2);
    cudaMalloc(&B, 256 * 640 * 2);
    cudaMemset(A, 0, 128 * 640 * 2);
    cudaMemset(B, 0, 256 * 640 * 2);
    cudaMalloc(&out, 8 * 64);
    run<32, 10>("BN=32 K=640", 1, 0, 128, A, B, out);
    run<32, 10>("BN=32 K=640", 1, 1, 128, A, B, out);
    run<32, 10>("BN=32 K=640 A 32 rows", 1, 1, 32, A, B, out);
    run<32, 10>("BN=32 K=640", 132, 1, 128, A, B, out);
    run<128, 6>("BN=128 K=384", 1, 0, 128, A, B, out);
    run<128, 6>("BN=128 K=384", 1, 1, 128, A, B, out);
    run<128, 6>("BN=128 K=384", 80, 1, 128, A, B, out);
    return 0;
}
