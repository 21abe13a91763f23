// tcgen05.mma issue rate microbenchmark (measurement aid): n back-to-back
// M=128 x N x K=16 bf16 MMAs from smem operands already resident, one CTA.
#include <cuda.h>
#include <cstdio>
#include "tc_common.cuh"
using namespace tbeam_dev;

template <int N>
__global__ void __launch_bounds__(128, 1) rate(int nmma, int nacc, unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* done = reinterpret_cast<uint64_t*>(smem + 64 * 1024 + 64 * 1024);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
    for (int i = threadIdx.x; i < 32 * 1024; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (threadIdx.x == 0) { mbar_init(done, 1); mbar_fence_init(); }
    if (threadIdx.x < 32) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = umma_idesc_bf16(128, N);
        const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 64 * 1024);
        const long long t0 = clock64();
        for (int j = 0; j < nmma; ++j) {
            const int kb = (j >> 2) % 4, k = j & 3;
            umma_bf16(tmem + (j % nacc) * N, umma_desc_sw128(a0 + kb * 16384 + 32 * k),
                      umma_desc_sw128(b0 + kb * 16384 + 32 * k), idesc, j >= nacc ? 1u : 0u);
        }
        const long long t1 = clock64();
        umma_commit(done);
        mbar_wait(done, 0);
        const long long t2 = clock64();
        out[0] = t1 - t0;
        out[1] = t2 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int N>
void run(int nmma, int nacc, unsigned long long* out) {
    const int smem = 1024 + 128 * 1024 + 64;
    cudaFuncSetAttribute(rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int r = 0; r < 3; ++r) rate<N><<<1, 128, smem>>>(nmma, nacc, out);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[2];
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("N=%3d mmas=%3d acc=%d: issue %6llu  done %6llu cycles  -> %5.1f cycles/MMA (%s)\n", N, nmma, nacc, h[0],
           h[1], (double)h[1] / nmma, cudaGetErrorString(e));
}

int main() {
    unsigned long long* out;
    cudaMalloc(&out, 16);
    run<32>(40, 1, out);
    run<32>(40, 4, out);
    run<64>(40, 4, out);
    run<128>(40, 2, out);
    run<256>(40, 1, out);
    run<32>(160, 4, out);
    run<256>(160, 1, out);
    return 0;
}
