// How accurate is an fp32 GEMM emulated on the tcgen05 tensor cores with
// split operands (measurement aid for the fp32 tensor-core path)?
//   x = x0 + x1 (+ x2), each part bf16 or tf32, products of the parts summed by
//   UMMA into fp32 TMEM accumulators -- one accumulator, or one per k-range
//   summed in fp64 by the epilogue -- against the fp64 product, next to the
//   CUDA-core FFMA schemes (sequential fp32; fp32 partial sums of 8 in fp64).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_2506_00185_b200/csrc -o split_mma split_mma.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>
#include "tc_common.cuh"
using namespace tbeam_dev;

constexpr int M = 128, N = 32, K = 640;

struct Maps {
    CUtensorMap a[3], b[3];
};

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// one CTA, 128 threads; per 128-B k-block all parts land, then every (ia, ib)
// pair issues its 4 K-steps into accumulator kb / kb_per_acc
template <bool TF32>
__global__ void __launch_bounds__(128, 1) split_gemm(const __grid_constant__ Maps maps, int npa, int npb,
                                                     const int* pairs, int npairs, int kb_per_acc, double* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    constexpr int AB = M * 128, BB = N * 128;
    constexpr int EPB = TF32 ? 32 : 64;  // elements per 128-B row
    constexpr int NK = K / EPB;
    uint8_t* sA = smem;
    uint8_t* sB = smem + 3 * AB;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + 3 * BB);
    uint64_t* done = full + 1;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
    const int nacc = (NK + kb_per_acc - 1) / kb_per_acc;
    if (threadIdx.x == 0) {
        mbar_init(full, 1);
        mbar_init(done, 1);
        mbar_fence_init();
    }
    if (threadIdx.x < 32) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t idesc = TF32 ? ((1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24))
                                : umma_idesc_bf16(M, N);
    for (int kb = 0; kb < NK; ++kb) {
        if (threadIdx.x == 0) {
            mbar_expect_tx(full, npa * AB + npb * BB);
            for (int p = 0; p < npa; ++p) tma_load_2d(sA + p * AB, &maps.a[p], full, kb * EPB, 0);
            for (int p = 0; p < npb; ++p) tma_load_2d(sB + p * BB, &maps.b[p], full, kb * EPB, 0);
        }
        if (threadIdx.x == 32) {
            mbar_wait(full, kb & 1);
            tc_fence_after();
            const int acc = kb / kb_per_acc;
            for (int q = 0; q < npairs; ++q) {
                const int ia = pairs[2 * q], ib = pairs[2 * q + 1];
                for (int k = 0; k < 4; ++k) {
                    const uint64_t da = umma_desc_sw128(smem_u32(sA + ia * AB) + 32 * k);
                    const uint64_t db = umma_desc_sw128(smem_u32(sB + ib * BB) + 32 * k);
                    const uint32_t accum = (kb % kb_per_acc != 0 || q != 0 || k != 0) ? 1u : 0u;
                    if (TF32) umma_tf32(tmem + acc * N, da, db, idesc, accum);
                    else umma_bf16(tmem + acc * N, da, db, idesc, accum);
                }
            }
            umma_commit(done);
            mbar_wait(done, kb & 1);
        }
        __syncthreads();
    }
    tc_fence_after();
    const int row = threadIdx.x;
    double s[N];
    for (int c = 0; c < N; ++c) s[c] = 0.0;
    for (int a = 0; a < nacc; ++a) {
        float v[32];
        tmem_ld32(tmem + ((threadIdx.x & ~31u) << 16) + a * N, v);
        for (int c = 0; c < N; ++c) s[c] += static_cast<double>(v[c]);
    }
    for (int c = 0; c < N; ++c) out[row * N + c] = s[c];
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

PFN_cuTensorMapEncodeTiled_v12000 enc_fn;
CUtensorMap mk(void* p, int rows, bool tf32) {
    CUtensorMap t;
    const int es = tf32 ? 4 : 2;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t str[1] = {(cuuint64_t)K * es};
    cuuint32_t box[2] = {(cuuint32_t)(128 / es), (cuuint32_t)rows};
    cuuint32_t el[2] = {1, 1};
    CUresult r = enc_fn(&t, tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, str,
                        box, el, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("tensor map error %d\n", (int)r);
    return t;
}

float bf(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
float tf(float x) {  // round to nearest tf32 (10 explicit mantissa bits)
    uint32_t u;
    memcpy(&u, &x, 4);
    u = (u + 0x1000u) & ~0x1FFFu;
    float y;
    memcpy(&y, &u, 4);
    return y;
}

struct Parts {
    std::vector<float> p[3];
};
Parts split(const std::vector<float>& x, int nparts, bool tf32) {
    Parts r;
    std::vector<float> rem = x;
    for (int q = 0; q < nparts; ++q) {
        r.p[q].resize(x.size());
        for (size_t i = 0; i < x.size(); ++i) {
            const float h = tf32 ? tf(rem[i]) : bf(rem[i]);
            r.p[q][i] = h;
            rem[i] -= h;  // exact (Sterbenz-style: h is a rounding of rem)
        }
    }
    return r;
}

int main() {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc_fn), cudaEnableDefault, &q);
    std::mt19937 g(1);
    std::normal_distribution<float> nd(0.f, 1.f);
    std::vector<float> A(M * K), B(N * K);
    for (auto& x : A) x = std::tanh(nd(g));               // z = tanh(enc + pred)
    for (auto& x : B) x = 4.0f * nd(g) / std::sqrt(float(K));  // W_out, logit scale 4
    std::vector<double> ref(M * N);
    double mag = 0;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
            double s = 0;
            for (int k = 0; k < K; ++k) s += double(A[i * K + k]) * double(B[j * K + k]);
            ref[i * N + j] = s;
            mag += std::fabs(s);
        }
    printf("mean |logit| %.3f\n", mag / (M * N));
    auto report = [&](const char* name, const std::vector<double>& got) {
        double mx = 0, ss = 0;
        for (int i = 0; i < M * N; ++i) {
            const double e = got[i] - ref[i];
            mx = std::fmax(mx, std::fabs(e));
            ss += e * e;
        }
        printf("%-46s max |err| %.3e  rms %.3e\n", name, mx, std::sqrt(ss / (M * N)));
    };
    {  // CUDA-core schemes emulated on the host
        std::vector<double> seq(M * N), f8(M * N);
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < N; ++j) {
                float s = 0;
                double d = 0;
                float p = 0;
                for (int k = 0; k < K; ++k) {
                    s = std::fmaf(A[i * K + k], B[j * K + k], s);
                    p = std::fmaf(A[i * K + k], B[j * K + k], p);
                    if (k % 8 == 7) d += p, p = 0;
                }
                seq[i * N + j] = s;
                f8[i * N + j] = d;
            }
        report("FFMA fp32 sequential", seq);
        report("FFMA partial sums of 8 in fp64", f8);
    }
    double* dout;
    cudaMalloc(&dout, sizeof(double) * M * N);
    int* dpairs;
    cudaMalloc(&dpairs, 64);
    void* dbuf[6];
    for (auto& p : dbuf) cudaMalloc(&p, M * K * 4);
    const int smem = 1024 + 3 * (M * 128 + N * 128) + 256;
    cudaFuncSetAttribute(split_gemm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(split_gemm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    auto run = [&](const char* name, bool tf32, int nparts, std::vector<int> pairs, int kb_per_acc) {
        Parts pa = split(A, nparts, tf32), pb = split(B, nparts, tf32);
        Maps maps;
        for (int p = 0; p < nparts; ++p) {
            if (tf32) {
                cudaMemcpy(dbuf[p], pa.p[p].data(), M * K * 4, cudaMemcpyHostToDevice);
                cudaMemcpy(dbuf[3 + p], pb.p[p].data(), N * K * 4, cudaMemcpyHostToDevice);
            } else {
                std::vector<__nv_bfloat16> ha(M * K), hb(N * K);
                for (int i = 0; i < M * K; ++i) ha[i] = __float2bfloat16_rn(pa.p[p][i]);
                for (int i = 0; i < N * K; ++i) hb[i] = __float2bfloat16_rn(pb.p[p][i]);
                cudaMemcpy(dbuf[p], ha.data(), M * K * 2, cudaMemcpyHostToDevice);
                cudaMemcpy(dbuf[3 + p], hb.data(), N * K * 2, cudaMemcpyHostToDevice);
            }
            maps.a[p] = mk(dbuf[p], M, tf32);
            maps.b[p] = mk(dbuf[3 + p], N, tf32);
        }
        cudaMemcpy(dpairs, pairs.data(), 4 * pairs.size(), cudaMemcpyHostToDevice);
        if (tf32) split_gemm<true><<<1, 128, smem>>>(maps, nparts, nparts, dpairs, pairs.size() / 2, kb_per_acc, dout);
        else split_gemm<false><<<1, 128, smem>>>(maps, nparts, nparts, dpairs, pairs.size() / 2, kb_per_acc, dout);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<double> got(M * N);
        cudaMemcpy(got.data(), dout, sizeof(double) * M * N, cudaMemcpyDeviceToHost);
        char lab[128];
        snprintf(lab, sizeof lab, "%s [acc per %d kb]%s", name, kb_per_acc, e == cudaSuccess ? "" : " ERROR");
        report(lab, got);
    };
    // pairs listed smallest magnitude first
    const std::vector<int> one = {0, 0};
    const std::vector<int> two3 = {1, 0, 0, 1, 0, 0};                    // x1y0 + x0y1 + x0y0
    const std::vector<int> three6 = {2, 0, 1, 1, 0, 2, 1, 0, 0, 1, 0, 0};  // + x2y0 x1y1 x0y2
    for (int kpa : {64, 4, 1}) {
        run("bf16 (1 part)", false, 1, one, kpa);
        run("bf16 x2 (3 products)", false, 2, two3, kpa);
        run("bf16 x3 (6 products)", false, 3, three6, kpa);
        run("tf32 (1 part)", true, 1, one, kpa == 1 ? 2 : kpa);
        run("tf32 x2 (3 products)", true, 2, two3, kpa == 1 ? 2 : kpa);
        run("tf32 x3 (6 products)", true, 3, three6, kpa == 1 ? 2 : kpa);
    }
    return 0;
}
