// filter.cu -- texture filtering on top of random-access decode (SURVEY.md 8(f) f2,
// PAPER.md:622-639): nearest, software bilinear (4 decodes) and trilinear (8 decodes), and
// stochastic filtering (U(-1/2,1/2) texel jitter, optional LOD jitter, one nearest decode).
// The decodes run in the tcgen05 decode kernel (query mode); these kernels only generate
// the queries and blend.  Product code.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "material.h"

namespace ntc {
cudaError_t decode_queries(const ntc_material* m, const ntc_query* q, int64_t n, uint16_t* out, int32_t* status,
                           cudaStream_t s);
ntc_status api_fail(ntc_status s, const char* msg);

__device__ __forceinline__ uint4 philox_f(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

// U(-1/2, 1/2) jitter, exact: (2(w >> 9) + 1) 2^-24 - 1/2
__device__ __forceinline__ double jitter(uint32_t w) { return (double)(2u * (w >> 9) + 1u) * 5.9604644775390625e-8 - 0.5; }

__device__ __forceinline__ ntc_query make_q(int x, int y, int m) {
    ntc_query q;
    q.x = (uint16_t)x;
    q.y = (uint16_t)y;
    q.mip = (uint8_t)m;
    q.material = 0;
    q.pad[0] = q.pad[1] = 0;
    return q;
}

// K queries per sample (+ blend weights): K = 1 (nearest / stochastic), 4 (bilinear), 8 (trilinear)
__global__ void filter_queries_kernel(const float* __restrict__ uvl, int64_t n, int mode, uint64_t seed, int W, int M,
                                      ntc_query* __restrict__ q, float* __restrict__ wts) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double u = uvl[3 * i], v = uvl[3 * i + 1];
    double lod = uvl[3 * i + 2];
    if (mode == 0 || mode >= 3) {
        double ju = 0.0, jv = 0.0;
        if (mode >= 3) {
            const uint4 r = philox_f(make_uint4((uint32_t)i, (uint32_t)((uint64_t)i >> 32), 0u, 0x46494C54u),
                                     make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
            ju = jitter(r.x);
            jv = jitter(r.y);
            if (mode == 4) lod += jitter(r.z);
        }
        const int m = min(max((int)floor(lod + 0.5), 0), M - 1), wm = W >> m;
        const int x = min(max((int)floor(u * wm + ju), 0), wm - 1), y = min(max((int)floor(v * wm + jv), 0), wm - 1);
        q[i] = make_q(x, y, m);
        return;
    }
    int mips[2];
    double mw[2];
    int nm;
    if (mode == 1) {
        mips[0] = min(max((int)floor(lod + 0.5), 0), M - 1);
        mw[0] = 1.0;
        nm = 1;
    } else {
        const double fl = floor(lod);
        mips[0] = min(max((int)fl, 0), M - 1);
        mips[1] = min(mips[0] + 1, M - 1);
        const double t = (lod >= M - 1 || lod < 0) ? 0.0 : lod - fl;
        mw[0] = 1.0 - t;
        mw[1] = t;
        nm = 2;
    }
    const int K = 4 * nm;
    for (int a = 0; a < nm; ++a) {
        const int m = mips[a], wm = W >> m;
        const double s = u * wm - 0.5, t = v * wm - 0.5;
        const double fs = floor(s), ft = floor(t);
        const double ax = s - fs, ay = t - ft;
        const int x0 = (int)fs, y0 = (int)ft;
        const double bw[4] = {(1 - ax) * (1 - ay), ax * (1 - ay), (1 - ax) * ay, ax * ay};
        for (int k = 0; k < 4; ++k) {
            const int x = min(max(x0 + (k & 1), 0), wm - 1), y = min(max(y0 + (k >> 1), 0), wm - 1);
            q[i * K + 4 * a + k] = make_q(x, y, m);
            wts[i * K + 4 * a + k] = (float)(mw[a] * bw[k]);
        }
    }
}

__global__ void filter_blend_kernel(const uint16_t* __restrict__ dec, const float* __restrict__ wts, int64_t n, int K,
                                    int c, uint16_t* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * c) return;
    const int64_t s = i / c;
    const int ch = (int)(i % c);
    float acc = 0.0f;
    for (int k = 0; k < K; ++k) acc += wts[s * K + k] * __half2float(__ushort_as_half(dec[(s * K + k) * c + ch]));
    out[i] = __half_as_ushort(__float2half_rn(acc));
}

static int taps_of(int mode) { return mode == 1 ? 4 : (mode == 2 ? 8 : 1); }

}  // namespace ntc

using namespace ntc;

extern "C" int64_t ntc_filter_scratch_bytes(int64_t n, int32_t mode, int32_t channels) {
    if (n < 0 || mode < 0 || mode > 4 || channels < 1 || channels > 16) return -1;
    const int K = taps_of(mode);
    int64_t b = n * K * (int64_t)sizeof(ntc_query);
    if (K > 1) b += n * K * (int64_t)sizeof(float) + n * K * channels * 2;
    return (b + 255) / 256 * 256;
}

extern "C" ntc_status ntc_filter_texels(const ntc_material* m, const float* uvl, int64_t n, int32_t mode,
                                        uint64_t seed, uint16_t* out, void* scratch, ntc_stream stream) {
    if (!m || n < 0 || mode < 0 || mode > 4) return api_fail(NTC_ERR_INVALID_ARGUMENT, "bad argument");
    if (n == 0) return NTC_OK;
    if (!uvl || !out || !scratch) return api_fail(NTC_ERR_INVALID_ARGUMENT, "NULL buffer");
    cudaStream_t st = (cudaStream_t)stream;
    const int K = taps_of(mode), c = m->d.channels;
    ntc_query* q = reinterpret_cast<ntc_query*>(scratch);
    float* wts = reinterpret_cast<float*>(q + n * K);
    uint16_t* dec = reinterpret_cast<uint16_t*>(wts + n * K);
    filter_queries_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(uvl, n, mode, seed, m->d.width, m->M, q, wts);
    cudaError_t e = decode_queries(m, q, n * K, K == 1 ? out : dec, nullptr, st);
    if (e == cudaSuccess && K > 1)
        filter_blend_kernel<<<(unsigned)((n * c + 255) / 256), 256, 0, st>>>(dec, wts, n, K, c, out);
    if (e == cudaSuccess) e = cudaGetLastError();
    return e == cudaSuccess ? NTC_OK : api_fail(NTC_ERR_CUDA, cudaGetErrorString(e));
}
