// Instruction-cache microbenchmark (measurement aid): does a kernel's code
// stay warm across launches, and how much intervening code evicts it?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o icache icache.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int N, int SALT>
__global__ void pad_kernel(unsigned* out, unsigned long long* t) {
    const unsigned long long t0 = clock64();
    unsigned x = clock(), y = x | 1u, z = y >> 3;
    unsigned x1 = x + 1 + SALT, x2 = x + 2, x3 = x + 3;
#pragma unroll
    for (int q = 0; q < N / 4; ++q) {
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z));
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x1) : "r"(y), "r"(z));
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x2) : "r"(y), "r"(z));
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x3) : "r"(y), "r"(z));
    }
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) {
        out[blockIdx.x] = x ^ x1 ^ x2 ^ x3;
        atomicAdd(t, t1 - t0);
    }
}

int main() {
    unsigned* out;
    unsigned long long* t;
    cudaMalloc(&out, 4096 * 4);
    cudaMalloc(&t, 8);
    auto run = [&](auto k, int blocks) {
        cudaMemset(t, 0, 8);
        k<<<blocks, 32>>>(out, t);
        cudaDeviceSynchronize();
        unsigned long long h;
        cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
        return (double)h / blocks;
    };
    const int B = 148;
    printf("A(3000) cold: %.0f cycles\n", run(pad_kernel<3000, 0>, B));
    printf("A(3000) again: %.0f\n", run(pad_kernel<3000, 0>, B));
    printf("A(3000) again: %.0f\n", run(pad_kernel<3000, 0>, B));
    for (int rep = 0; rep < 2; ++rep) {
        run(pad_kernel<2000, 1>, B);
        printf("after B(2000): A %.0f\n", run(pad_kernel<3000, 0>, B));
        run(pad_kernel<6000, 2>, B);
        printf("after B(6000): A %.0f\n", run(pad_kernel<3000, 0>, B));
        run(pad_kernel<12000, 3>, B);
        printf("after B(12000): A %.0f\n", run(pad_kernel<3000, 0>, B));
    }
    printf("B(12000) cold-ish: %.0f\n", run(pad_kernel<12000, 4>, B));
    printf("B(12000) again: %.0f\n", run(pad_kernel<12000, 4>, B));
    return 0;
}
