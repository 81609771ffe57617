// mma_probe.cu -- micro-probe of tcgen05.mma on B200 (profiling helper, not product code):
// (1) issue -> mbarrier-completion latency of short MMA groups (SS operands, and A in TMEM);
// (2) correctness of the A-from-TMEM layout assumption (lane = row, column c = k 2c, 2c+1).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_probe tools/mma_probe.cu
#include <cuda_fp16.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2305_17105_b200/csrc/ptx.cuh"

using namespace ntc;

__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                           uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

// A: 128 x 64 fp16 (row-major, host), B: 64 x 64 fp16 (n-major rows of k). out: D_ss, D_ts [128][64]
__global__ void probe(const __half* A, const __half* B, float* dss, float* dts, long long* lat, int reps) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tm;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    uint8_t* sa = smem;          // 16 KB
    uint8_t* sb = smem + 16384;  // 8 KB
    for (int i = tid; i < 128 * 64; i += blockDim.x) {
        const int r = i / 64, k = i % 64;
        *reinterpret_cast<__half*>(sa + sw128_offset(r, k)) = A[i];
    }
    for (int i = tid; i < 64 * 64; i += blockDim.x) {
        const int r = i / 64, k = i % 64;
        *reinterpret_cast<__half*>(sb + sw128_offset(r, k)) = B[i];
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(&tm, 256);
        tmem_relinquish();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t t = tm;
    const uint32_t d1 = t, d2 = t + 64, ta = t + 128;  // A in TMEM at columns [128, 160)
    // A row `tid` into TMEM: 32 columns, column c = (A[r][2c], A[r][2c+1])
    {
        uint32_t r[32];
        for (int c = 0; c < 32; ++c) {
            __half2 h = __halves2half2(A[tid * 64 + 2 * c], A[tid * 64 + 2 * c + 1]);
            r[c] = *reinterpret_cast<uint32_t*>(&h);
        }
        tmem_st32(ta + ((uint32_t)(warp * 32) << 16), r);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint64_t adesc = umma_desc_k_sw128(smem_u32(sa)), bdesc = umma_desc_k_sw128(smem_u32(sb));
    const uint32_t id = idesc_f16(128, 64);
    uint32_t ph = 0;
    if (tid == 0) {
        for (int k = 0; k < 4; ++k) mma_f16_ss(d1, adesc + 2 * k, bdesc + 2 * k, id, k > 0);
        for (int k = 0; k < 4; ++k) mma_f16_ts(d2, ta + 8 * k, bdesc + 2 * k, id, k > 0);
        mma_commit(&bar);
    }
    mbar_wait(&bar, ph);
    ph ^= 1;
    tc_fence_after();
    {
        uint32_t r[32];
        for (int h = 0; h < 2; ++h) {
            tmem_ld32(d1 + ((uint32_t)(warp * 32) << 16) + 32 * h, r);
            tmem_wait_ld();
            for (int c = 0; c < 32; ++c) dss[tid * 64 + 32 * h + c] = __uint_as_float(r[c]);
            tmem_ld32(d2 + ((uint32_t)(warp * 32) << 16) + 32 * h, r);
            tmem_wait_ld();
            for (int c = 0; c < 32; ++c) dts[tid * 64 + 32 * h + c] = __uint_as_float(r[c]);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // latency of groups: 4 SS (N64), 5 SS (N64), 4 TS (N64), 1 SS (N64), 4 SS (N16)
    if (tid == 0) {
        for (int v = 0; v < 8; ++v) {
            long long best = 1LL << 60, sum = 0;
            for (int it = 0; it < reps; ++it) {
                const long long c0 = clock64();
                if (v == 0) for (int k = 0; k < 4; ++k) mma_f16_ss(d1, adesc + 2 * k, bdesc + 2 * k, id, k > 0);
                if (v == 1) for (int k = 0; k < 5; ++k) mma_f16_ss(d1, adesc + 2 * (k & 3), bdesc + 2 * (k & 3), id, k > 0);
                if (v == 2) for (int k = 0; k < 4; ++k) mma_f16_ts(d2, ta + 8 * k, bdesc + 2 * k, id, k > 0);
                if (v == 3) mma_f16_ss(d1, adesc, bdesc, id, 0);
                if (v == 4) for (int k = 0; k < 4; ++k) mma_f16_ss(d1, adesc + 2 * k, bdesc + 2 * k, idesc_f16(128, 16), k > 0);
                if (v == 5) for (int k = 0; k < 8; ++k) mma_f16_ss((k & 1) ? d2 : d1, adesc + 2 * (k >> 1), bdesc + 2 * (k >> 1), id, k > 1);
                if (v == 6) for (int k = 0; k < 16; ++k) mma_f16_ss(t + 32 * (k & 3), adesc + 2 * (k >> 2), bdesc + 2 * (k >> 2), idesc_f16(128, 32), k > 3);
                if (v == 7) for (int k = 0; k < 16; ++k) mma_f16_ss(d1, adesc + 2 * (k & 3), bdesc + 2 * (k & 3), id, k > 0);
                mma_commit(&bar);
                mbar_wait(&bar, ph);
                ph ^= 1;
                const long long c1 = clock64();
                best = min(best, c1 - c0);
                sum += c1 - c0;
            }
            lat[2 * v] = best;
            lat[2 * v + 1] = sum / reps;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(t, 256);
}

int main() {
    std::vector<__half> A(128 * 64), B(64 * 64);
    srand(1);
    for (auto& v : A) v = __float2half((rand() % 17 - 8) / 8.0f);
    for (auto& v : B) v = __float2half((rand() % 17 - 8) / 16.0f);
    __half *dA, *dB;
    float *dss, *dts;
    long long* dlat;
    cudaMalloc(&dA, A.size() * 2);
    cudaMalloc(&dB, B.size() * 2);
    cudaMalloc(&dss, 128 * 64 * 4);
    cudaMalloc(&dts, 128 * 64 * 4);
    cudaMalloc(&dlat, 16 * 8);
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    probe<<<1, 128, 32768>>>(dA, dB, dss, dts, dlat, 200);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
    }
    std::vector<float> ss(128 * 64), ts(128 * 64);
    long long lat[16];
    cudaMemcpy(ss.data(), dss, ss.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(ts.data(), dts, ts.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(lat, dlat, sizeof lat, cudaMemcpyDeviceToHost);
    double maxref = 0, errss = 0, errts = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
            double r = 0;
            for (int k = 0; k < 64; ++k) r += (double)__half2float(A[m * 64 + k]) * (double)__half2float(B[n * 64 + k]);
            maxref = fmax(maxref, fabs(r));
            errss = fmax(errss, fabs(ss[m * 64 + n] - r));
            errts = fmax(errts, fabs(ts[m * 64 + n] - r));
        }
    printf("max|ref| %.3f  max err SS %.3g  TS %.3g\n", maxref, errss, errts);
    const char* names[8] = {"4xSS N64 K16", "5xSS N64 K16", "4xTS N64 K16", "1xSS N64 K16", "4xSS N16 K16",
                            "2 chains x4 N64", "4 chains x4 N32", "16 dep N64"};
    for (int v = 0; v < 8; ++v) printf("%-14s latency min %lld avg %lld cycles\n", names[v], lat[2 * v], lat[2 * v + 1]);
    return 0;
}
