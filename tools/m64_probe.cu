// m64_probe.cu -- where does a cta_group::1 M=64 tcgen05.mma put its 64 accumulator rows in
// TMEM?  (profiling helper, not product code).  Fills 16 TMEM columns of all 128 lanes with
// a sentinel, runs one M=64 N=16 K=16 MMA (row r of A = r+1 in column 0, B = identity-ish),
// reads the 128 lanes back and prints which lanes hold which row.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o m64_probe tools/m64_probe.cu
#include <cuda_fp16.h>

#include <cstdio>
#include <vector>

#include "../paper_2305_17105_b200/csrc/ptx.cuh"

using namespace ntc;

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

__global__ void probe(float* out, int m_rows, int lane_base) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tm;
    const int tid = threadIdx.x, warp = tid / 32;
    uint8_t* sa = smem;          // A: 128 rows x 64 K (only K 0..15 used), SW128
    uint8_t* sb = smem + 16384;  // B: 16 rows (N) x 64 K
    for (int i = tid; i < 128 * 64; i += blockDim.x) {
        const int r = i / 64, k = i % 64;
        *reinterpret_cast<__half*>(sa + sw128_offset(r, k)) = __float2half(k == 0 ? (float)(r + 1) : 0.0f);
    }
    for (int i = tid; i < 16 * 64; i += blockDim.x) {
        const int n = i / 64, k = i % 64;
        *reinterpret_cast<__half*>(sb + sw128_offset(n, k)) = __float2half(k == 0 ? (float)(n + 1) * 1000.0f : 0.0f);
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(&tm, 32);
        tmem_relinquish();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t t = tm;
    {
        uint32_t s[16];
        for (int c = 0; c < 16; ++c) s[c] = __float_as_uint(-1.0f);
        tmem_st16(t + ((uint32_t)(warp * 32) << 16), s);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        mma_f16_ss(t + ((uint32_t)lane_base << 16), umma_desc_k_sw128(smem_u32(sa)), umma_desc_k_sw128(smem_u32(sb)),
                   idesc_f16(m_rows, 16), 0);
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    uint32_t r[16];
    tmem_ld16(t + ((uint32_t)(warp * 32) << 16), r);
    tmem_wait_ld();
    for (int c = 0; c < 16; ++c) out[tid * 16 + c] = __uint_as_float(r[c]);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(t, 32);
}

int main() {
    float* d;
    cudaMalloc(&d, 128 * 16 * 4);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    for (int m : {64, 64}) {
        static int call = 0;
        const int lb = call++ == 0 ? 0 : 16;
        probe<<<1, 128, 32768>>>(d, m, lb);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("M=%d error %s\n", m, cudaGetErrorString(e));
            return 1;
        }
        std::vector<float> h(128 * 16);
        cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
        printf("M=%d lane_base=%d: lane -> (col0 / 1000 = A row + 1, col1 / 2000 = A row + 1)\n", m, lb);
        for (int lane = 0; lane < 128; ++lane) {
            printf("%3d:%7.1f %7.1f%s", lane, h[lane * 16], h[lane * 16 + 1], (lane % 4 == 3) ? "\n" : " | ");
        }
    }
    return 0;
}
