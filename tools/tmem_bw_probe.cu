// tmem_bw_probe.cu -- micro-probe (profiling helper, not product code): per-SM throughput of
// tcgen05.ld (TMEM -> registers) and tcgen05.st for the load shapes the decode epilogue uses,
// with 4 / 8 / 16 warps per CTA and one CTA per SM on all SMs; plus the TMEM layout of a
// kind::f16 MMA with an fp16 accumulator (idesc bit 4 = 0), raw words of row 0.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tmem_bw_probe tools/tmem_bw_probe.cu
#include <cuda_fp16.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2305_17105_b200/csrc/ptx.cuh"

using namespace ntc;

__device__ __forceinline__ void ld_x64(uint32_t taddr, uint32_t (&r)[64]) {
    tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
    tmem_ld32(taddr + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

// 16 columns of 16-bit data packed two per register (.pack::16b): reads columns c, c+1 into one reg
__device__ __forceinline__ void tmem_ld16_pack(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
}

// mode 0: x16 + wait; 1: 4 x x16 then wait; 2: x32 + wait; 3: 2 x x32 then wait; 4: x16 pack::16b + wait;
// 5: st x16 + wait::st; 6: STS.128 (smem reference)
__global__ void bw(int mode, int iters, unsigned long long* cyc, uint32_t* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tm;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        tmem_alloc(&tm, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t t = tm + ((uint32_t)((warp & 3) * 32) << 16);
    const int colbase = (warp >> 2) * 128;  // warps of the same quarter use different columns
    uint32_t acc = 0;
    __syncthreads();
    const unsigned long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const uint32_t col = (uint32_t)(colbase + ((it * 64) & 127));
        if (mode == 0) {
            uint32_t r[16];
            tmem_ld16(t + col, r);
            tmem_wait_ld_r16(r);
            for (int i = 0; i < 16; ++i) acc ^= r[i];
        } else if (mode == 1) {
            uint32_t r[4][16];
            for (int j = 0; j < 4; ++j) tmem_ld16(t + col + 16 * j, r[j]);
            tmem_wait_ld();
            for (int j = 0; j < 4; ++j)
                for (int i = 0; i < 16; ++i) acc ^= r[j][i];
        } else if (mode == 2) {
            uint32_t r[32];
            tmem_ld32(t + col, r);
            tmem_wait_ld();
            for (int i = 0; i < 32; ++i) acc ^= r[i];
        } else if (mode == 3) {
            uint32_t r[64];
            ld_x64(t + col, r);
            tmem_wait_ld();
            for (int i = 0; i < 64; ++i) acc ^= r[i];
        } else if (mode == 4) {
            uint32_t r[8];
            tmem_ld16_pack(t + col, r);
            tmem_wait_ld();
            for (int i = 0; i < 8; ++i) acc ^= r[i];
        } else if (mode == 5) {
            uint32_t r[16];
            for (int i = 0; i < 16; ++i) r[i] = acc + i;
            tmem_st16(t + col, r);
            tmem_wait_st();
            acc += 1;
        } else {
            const uint32_t a = smem_u32(smem) + (uint32_t)threadIdx.x * 16u + (uint32_t)((it & 3) * 8192);
            for (int j = 0; j < 4; ++j) sts128(a + 2048u * j, acc, acc + 1, acc + 2, acc + j);
            acc += 3;
        }
    }
    const unsigned long long c1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
    if (acc == 0x12345678u) sink[0] = acc;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(tm, 512);
}

// fp16-accumulator MMA: D (f16) = A . B^T, raw TMEM words of rows 0 and 1, columns 0..63
__global__ void f16acc(const __half* A, const __half* B, uint32_t* raw, int dtype_f32) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tm;
    const int tid = threadIdx.x, warp = tid / 32;
    uint8_t* sa = smem;
    uint8_t* sb = smem + 16384;
    for (int i = tid; i < 128 * 64; i += blockDim.x)
        *reinterpret_cast<__half*>(sa + sw128_offset(i / 64, i % 64)) = A[i];
    for (int i = tid; i < 64 * 64; i += blockDim.x)
        *reinterpret_cast<__half*>(sb + sw128_offset(i / 64, i % 64)) = B[i];
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(&tm, 128);
        tmem_relinquish();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t t = tm;
    // zero the 64 columns first so untouched columns read as 0
    {
        uint32_t z[16];
        for (int i = 0; i < 16; ++i) z[i] = 0u;
        for (int j = 0; j < 4; ++j) tmem_st16(t + ((uint32_t)(warp * 32) << 16) + 16 * j, z);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t id = dtype_f32 ? idesc_f16(128, 64) : (idesc_f16(128, 64) & ~(3u << 4));
    if (tid == 0) {
        const uint64_t ad = umma_desc_k_sw128(smem_u32(sa)), bd = umma_desc_k_sw128(smem_u32(sb));
        for (int k = 0; k < 4; ++k) mma_f16_ss(t, ad + 2 * k, bd + 2 * k, id, k > 0);
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    uint32_t r[32];
    for (int h = 0; h < 2; ++h) {
        tmem_ld32(t + ((uint32_t)(warp * 32) << 16) + 32 * h, r);
        tmem_wait_ld();
        for (int c = 0; c < 32; ++c) raw[tid * 64 + 32 * h + c] = r[c];
    }
    uint32_t p[8];
    tmem_ld16_pack(t + ((uint32_t)(warp * 32) << 16), p);
    tmem_wait_ld();
    for (int c = 0; c < 8; ++c) raw[128 * 64 + tid * 8 + c] = p[c];
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(t, 128);
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* dc;
    uint32_t* ds;
    cudaMalloc(&dc, nsm * 8);
    cudaMalloc(&ds, 4);
    cudaFuncSetAttribute(bw, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 8192 + 1024);
    const char* names[7] = {"ld x16+wait", "4x ld x16, wait", "ld x32+wait", "2x ld x32, wait", "ld x16 pack16b",
                            "st x16+wait", "STS.128 x4"};
    const int bytes_per_it[7] = {16 * 4, 64 * 4, 32 * 4, 64 * 4, 16 * 4, 16 * 4, 64};
    for (int mode = 0; mode < 7; ++mode)
        for (int nw : {1, 4, 8, 16}) {
            const int iters = 4096;
            bw<<<nsm, nw * 32, 8 * 8192 + 1024>>>(mode, iters, dc, ds);
            bw<<<nsm, nw * 32, 8 * 8192 + 1024>>>(mode, iters, dc, ds);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("error %s\n", cudaGetErrorString(e));
                return 1;
            }
            std::vector<unsigned long long> c(nsm);
            cudaMemcpy(c.data(), dc, nsm * 8, cudaMemcpyDeviceToHost);
            unsigned long long mx = 0, sum = 0;
            for (auto v : c) mx = v > mx ? v : mx, sum += v;
            const double bytes = (double)nw * 32 * bytes_per_it[mode] * iters;
            printf("%-18s warps %2d: %8.1f B/cyc/SM (avg cyc %llu, %.1f cyc per warp-op)\n", names[mode], nw,
                   bytes / ((double)sum / nsm), sum / nsm, (double)(sum / nsm) / iters);
        }
    // fp16-accumulator layout
    std::vector<__half> A(128 * 64), B(64 * 64);
    srand(1);
    for (auto& v : A) v = __float2half((rand() % 17 - 8) / 8.0f);
    for (auto& v : B) v = __float2half((rand() % 17 - 8) / 16.0f);
    __half *dA, *dB;
    uint32_t* draw;
    cudaMalloc(&dA, A.size() * 2);
    cudaMalloc(&dB, B.size() * 2);
    cudaMalloc(&draw, (128 * 64 + 128 * 8) * 4);
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(f16acc, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    for (int f32 = 0; f32 < 2; ++f32) {
        cudaMemset(draw, 0, (128 * 64 + 128 * 8) * 4);
        f16acc<<<1, 128, 32768>>>(dA, dB, draw, f32);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("f16acc error %s\n", cudaGetErrorString(e));
            return 1;
        }
        std::vector<uint32_t> raw(128 * 64 + 128 * 8);
        cudaMemcpy(raw.data(), draw, raw.size() * 4, cudaMemcpyDeviceToHost);
        printf("accumulator %s: reference row 0 n=0..7:", f32 ? "f32" : "f16");
        for (int n = 0; n < 8; ++n) {
            double r = 0;
            for (int k = 0; k < 64; ++k) r += (double)__half2float(A[k]) * (double)__half2float(B[n * 64 + k]);
            printf(" %.4f", r);
        }
        printf("\n  raw words row 0 col 0..15:");
        for (int cc = 0; cc < 16; ++cc) printf(" %08x", raw[cc]);
        printf("\n  raw words row 0 col 32..39:");
        for (int cc = 32; cc < 40; ++cc) printf(" %08x", raw[cc]);
        printf("\n  pack::16b row 0 words 0..7:");
        for (int cc = 0; cc < 8; ++cc) printf(" %08x", raw[128 * 64 + cc]);
        printf("\n  as halves (lo, hi) of col 0..3:");
        for (int cc = 0; cc < 4; ++cc) {
            __half_raw lo, hi;
            lo.x = (unsigned short)(raw[cc] & 0xFFFF);
            hi.x = (unsigned short)(raw[cc] >> 16);
            printf(" (%.4f, %.4f)", __half2float(__half(lo)), __half2float(__half(hi)));
        }
        printf("\n");
    }
    return 0;
}
