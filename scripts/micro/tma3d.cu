// 3-D "all k-blocks in one box" TMA microbenchmark + correctness check
// (measurement aid).  View a row-major [rows][K] bf16 matrix as
// {64, rows, K/64} with strides {pitch, 128 B}: one box {64, R, nk} lands as
// nk consecutive [R][64] k-block tiles (128-B swizzled), i.e. the GEMM's
// stage layout for every k-block at once.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <vector>
#include "tc_common.cuh"
using namespace tbeam_dev;

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
        ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z) : "memory");
}

template <int R, int NK>
__global__ void k3(const __grid_constant__ CUtensorMap ta, int nbox, unsigned long long* out, unsigned* chk) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + NK * 128 * 128);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_fence_init();
    }
    __syncthreads();
    const long long t0 = clock64();
    if (threadIdx.x == 0) {
        mbar_expect_tx(bar, nbox * R * 128 * NK);
        for (int i = 0; i < nbox; ++i) tma_load_3d(smem + i * R * 128, &ta, bar, 0, R * i, 0);
    }
    mbar_wait(bar, 0);
    const long long t1 = clock64() - t0;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1;
    // check: k-block kb, row r, col c (unswizzled: 16-B chunk j of row r lives at chunk j ^ (r & 7))
    if (blockIdx.x == 0)
        for (int e = threadIdx.x; e < NK * nbox * R * 64; e += blockDim.x) {
            const int kb = e / (nbox * R * 64), rem = e % (nbox * R * 64), r = rem / 64, c = rem % 64;
            const int chunk = (c / 8) ^ (r & 7);
            const __nv_bfloat16* p = reinterpret_cast<const __nv_bfloat16*>(smem + (size_t)kb * 0 + 0);
            (void)p;
            // box i rows land at smem + i*R*128 ... + kb * (nbox*R*128)?  (dims order: x=64, y=rows, z=kb)
            const uint8_t* row = smem + ((size_t)kb * nbox * R + r) * 128;
            const __nv_bfloat16 v = reinterpret_cast<const __nv_bfloat16*>(row + chunk * 16)[c % 8];
            const float want = (float)((r * 7 + (kb * 64 + c) * 3) % 251);
            if (__bfloat162float(v) != want) atomicAdd(chk, 1u);
        }
}

PFN_cuTensorMapEncodeTiled_v12000 enc_fn;
int main() {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc_fn), cudaEnableDefault, &q);
    const int rows = 128, K = 640, pitch = 640;
    std::vector<__nv_bfloat16> h(rows * pitch);
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < K; ++c) h[r * pitch + c] = __float2bfloat16((float)((r * 7 + c * 3) % 251));
    void* A;
    cudaMalloc(&A, h.size() * 2);
    cudaMemcpy(A, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    unsigned long long* out;
    unsigned* chk;
    cudaMalloc(&out, 64);
    cudaMalloc(&chk, 4);
    auto test = [&](auto kern, int R, int nbox, const char* name) {
        CUtensorMap t;
        cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(K / 64)};
        cuuint64_t str[2] = {(cuuint64_t)pitch * 2, 128};
        cuuint32_t box[3] = {64, (cuuint32_t)R, 10};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult rc = enc_fn(&t, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, A, dims, str, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        cudaMemset(chk, 0, 4);
        const int smem = 1024 + 10 * 128 * 128 + 64;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int rep = 0; rep < 3; ++rep) kern<<<1, 128, smem>>>(t, nbox, out, chk);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long c;
        unsigned bad;
        cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(&bad, chk, 4, cudaMemcpyDeviceToHost);
        printf("%-28s encode=%d cycles=%llu mismatches=%u (%s)\n", name, (int)rc, c, bad, cudaGetErrorString(e));
    };
    test(k3<128, 10>, 128, 1, "box{64,128,10} x1");
    test(k3<32, 10>, 32, 2, "box{64,32,10} x2 (64 rows)");
    test(k3<32, 10>, 32, 4, "box{64,32,10} x4 (128 rows)");
    test(k3<64, 10>, 64, 1, "box{64,64,10} x1");
    return 0;
}
