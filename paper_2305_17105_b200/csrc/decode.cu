// decode.cu -- per-texel NTC decode on sm_100a (tcgen05 + TMEM), product code.
//
// One persistent CTA per SM, NWG = 4 warpgroups.  Each warpgroup owns a pipeline of
// 128-texel tiles (TMEM lane r <-> texel r <-> thread r of the warpgroup):
//   a1-a4  every thread assembles its texel's fp16 input row X (G0 2x2 gather, G1 bilinear,
//          PE, LOD, constant 1 for the folded bias b1) and stores it into a K-major,
//          128B-swizzled SMEM tile;
//   a5     one elected thread issues tcgen05.mma  D1[tmem] = X * W1^T  (M=128, N=64);
//   a5/a6  tcgen05.ld D1 -> +b, hardGELU -> fp16 -> SMEM (A operand of the next layer);
//   a7     D3 = H2 * W3^T (N=16) -> +b3, clamp [0,1] -> fp16 -> global (y, x, ch).
// The whole MLP weight set lives in SMEM for the CTA's lifetime (one copy per SM).
#include <cuda_fp16.h>

#include "common.cuh"
#include "ptx.cuh"

namespace ntc {

// ------------------------------------------------------------------ addressing (a1)
// R1/R2/R3: u = (x + 1/2) r / w_m - 1/2 (exact in fp32: r / w_m is a power of two),
// taps (i, j), (i+1, j), (i, j+1), (i+1, j+1) clamped to the grid.
struct Taps {
    int32_t j;
    int32_t x0[2], y0[2];  // G0 tap columns / rows
    int32_t x1[2], y1[2];  // G1 tap columns / rows
    float fx, fy;          // G1 fractional offsets (dyadic, exact)
};

__device__ __forceinline__ void address(const DecodeParams& p, int m, int x, int y, Taps& t) {
    const int j = p.level_of[m];
    const int r0 = p.lv[j].r0, r1 = p.lv[j].r1;
    const float wm = (float)(p.W >> m);
    t.j = j;
    {
        const float s = (float)r0 / wm;
        const float u = ((float)x + 0.5f) * s - 0.5f, v = ((float)y + 0.5f) * s - 0.5f;
        const int i = (int)floorf(u), k = (int)floorf(v);
        t.x0[0] = min(max(i, 0), r0 - 1);
        t.x0[1] = min(max(i + 1, 0), r0 - 1);
        t.y0[0] = min(max(k, 0), r0 - 1);
        t.y0[1] = min(max(k + 1, 0), r0 - 1);
    }
    {
        const float s = (float)r1 / wm;
        const float u = ((float)x + 0.5f) * s - 0.5f, v = ((float)y + 0.5f) * s - 0.5f;
        const float fu = floorf(u), fv = floorf(v);
        const int i = (int)fu, k = (int)fv;
        t.fx = u - fu;
        t.fy = v - fv;
        t.x1[0] = min(max(i, 0), r1 - 1);
        t.x1[1] = min(max(i + 1, 0), r1 - 1);
        t.y1[0] = min(max(k, 0), r1 - 1);
        t.y1[1] = min(max(k + 1, 0), r1 - 1);
    }
}

// ------------------------------------------------------------------ packed cells
template <int BYTES>
struct Cell {
    uint32_t w[BYTES >= 4 ? BYTES / 4 : 1];
};

template <int BYTES>
__device__ __forceinline__ Cell<BYTES> load_cell(const uint8_t* base, int64_t idx) {
    Cell<BYTES> c;
    if constexpr (BYTES == 1) {
        c.w[0] = __ldg(base + idx);
    } else if constexpr (BYTES == 2) {
        c.w[0] = __ldg(reinterpret_cast<const uint16_t*>(base) + idx);
    } else if constexpr (BYTES == 4) {
        c.w[0] = __ldg(reinterpret_cast<const uint32_t*>(base) + idx);
    } else if constexpr (BYTES == 8) {
        uint2 v = __ldg(reinterpret_cast<const uint2*>(base) + idx);
        c.w[0] = v.x;
        c.w[1] = v.y;
    } else {
        uint4 v = __ldg(reinterpret_cast<const uint4*>(base) + idx);
        c.w[0] = v.x;
        c.w[1] = v.y;
        c.w[2] = v.z;
        c.w[3] = v.w;
    }
    return c;
}

template <int B, int BYTES>
__device__ __forceinline__ uint32_t code_of(const Cell<BYTES>& c, int ch) {
    const int bit = ch * B;
    return (c.w[bit >> 5] >> (bit & 31)) & ((1u << B) - 1u);
}

// dequantise two codes to a half2 (idx * Q, idx = code - (N/2 - 1)):
// half(0x6400 | code) = 1024 + code; one HFMA2 maps it to (code - N/2 + 1) / N exactly.
template <int B>
__device__ __forceinline__ uint32_t dequant_pair(uint32_t lo, uint32_t hi) {
    constexpr float Q = 1.0f / (float)(1 << B);
    constexpr float OFF = (float)((1 << B) / 2 - 1);
    const uint32_t v = lo | (hi << 16) | 0x64006400u;
    const __half2 s = __float2half2_rn(Q);
    const __half2 o = __float2half2_rn(-(1024.0f + OFF) * Q);
    __half2 r = __hfma2(*reinterpret_cast<const __half2*>(&v), s, o);
    return *reinterpret_cast<uint32_t*>(&r);
}

__device__ __forceinline__ float code_f32(uint32_t code) {
    return __uint_as_float(0x4B000000u | code) - 8388608.0f;  // exact integer -> float
}

// ------------------------------------------------------------------ input assembly (a2-a4)
// X = [G0 taps (tap-major, channel-minor) | bilinear G1 | PE_x(6) | PE_y(6) | LOD | 1 | 0...]
// as K1W half2 words (R4; the trailing 1 multiplies the b1 column of the W1 image).
template <class P>
__device__ __forceinline__ void assemble_row(const DecodeParams& p, const uint32_t* s_pe, int m, int x, int y,
                                             uint32_t (&w)[P::K1W], int32_t* dbg_addr) {
    Taps t;
    address(p, m, x, y, t);
    const LevelGeom g = p.lv[t.j];
    const uint8_t* g0 = p.grids + g.off0;
    const uint8_t* g1 = p.grids + g.off1;
    // G0: four unfiltered taps ("learned interpolation")
#pragma unroll
    for (int tp = 0; tp < 4; ++tp) {
        const int cx = t.x0[tp & 1], cy = t.y0[tp >> 1];
        const Cell<P::CELL0> c = load_cell<P::CELL0>(g0, (int64_t)cy * g.r0 + cx);
#pragma unroll
        for (int k = 0; k < P::C0 / 2; ++k)
            w[tp * (P::C0 / 2) + k] = dequant_pair<P::B0>(code_of<P::B0>(c, 2 * k), code_of<P::B0>(c, 2 * k + 1));
    }
    // G1: bilinear; sums of dyadic products, exact in fp32, rounded once
    {
        Cell<P::CELL1> c[4];
#pragma unroll
        for (int tp = 0; tp < 4; ++tp)
            c[tp] = load_cell<P::CELL1>(g1, (int64_t)t.y1[tp >> 1] * g.r1 + t.x1[tp & 1]);
        const float wt[4] = {(1.0f - t.fx) * (1.0f - t.fy), t.fx * (1.0f - t.fy), (1.0f - t.fx) * t.fy,
                             t.fx * t.fy};
        constexpr float Q = 1.0f / (float)(1 << P::B1);
        constexpr float OFFQ = (float)((1 << P::B1) / 2 - 1) / (float)(1 << P::B1);
#pragma unroll
        for (int k = 0; k < P::C1 / 2; ++k) {
            float v[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                float a = wt[0] * code_f32(code_of<P::B1>(c[0], 2 * k + e));
                a = fmaf(wt[1], code_f32(code_of<P::B1>(c[1], 2 * k + e)), a);
                a = fmaf(wt[2], code_f32(code_of<P::B1>(c[2], 2 * k + e)), a);
                a = fmaf(wt[3], code_f32(code_of<P::B1>(c[3], 2 * k + e)), a);
                v[e] = fmaf(a, Q, -OFFQ);
            }
            w[2 * P::C0 + k] = pack_half2(v[0], v[1]);
        }
    }
    // PE from the 8-entry per-axis table, LOD + bias one
    constexpr int PEW = (4 * P::C0 + P::C1) / 2;
    const uint4 px = *reinterpret_cast<const uint4*>(s_pe + 4 * (x & 7));
    const uint4 py = *reinterpret_cast<const uint4*>(s_pe + 4 * (y & 7));
    w[PEW + 0] = px.x;
    w[PEW + 1] = px.y;
    w[PEW + 2] = px.z;
    w[PEW + 3] = py.x;
    w[PEW + 4] = py.y;
    w[PEW + 5] = py.z;
    w[PEW + 6] = p.lod_word[m];
#pragma unroll
    for (int k = PEW + 7; k < P::K1W; ++k) w[k] = 0u;
    if (dbg_addr) {
        dbg_addr[0] = t.j;
        for (int tp = 0; tp < 4; ++tp) {
            dbg_addr[1 + 2 * tp] = t.x0[tp & 1];
            dbg_addr[2 + 2 * tp] = t.y0[tp >> 1];
            dbg_addr[9 + 2 * tp] = t.x1[tp & 1];
            dbg_addr[10 + 2 * tp] = t.y1[tp >> 1];
        }
    }
}

// store NW half2 words of row `row` into a K-major SW128 tile of 128 rows
template <int NW>
__device__ __forceinline__ void store_row(uint32_t tile, int row, const uint32_t* w) {
#pragma unroll
    for (int c = 0; c < NW / 4; ++c) {
        const uint32_t addr = tile + (uint32_t)(c >> 3) * (128u * 128u) + (uint32_t)row * 128u +
                              ((uint32_t)((c & 7) ^ (row & 7)) << 4);
        sts128(addr, w[4 * c + 0], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
    }
}

// hardGELU = z * sat(z/3 + 1/2)
__device__ __forceinline__ float hardgelu(float z) { return z * __saturatef(fmaf(z, 1.0f / 3.0f, 0.5f)); }

// TMEM accumulator columns [0, 64) of this thread's lane -> +bias -> hardGELU -> 32 half2
template <int LAYER>
__device__ __forceinline__ void epilogue_hidden(const DecodeParams& p, uint32_t taddr, uint32_t (&h)[32]) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        uint32_t r[32];
        tmem_ld32(taddr + 32 * half, r);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            float z0 = __uint_as_float(r[2 * i]), z1 = __uint_as_float(r[2 * i + 1]);
            if constexpr (LAYER == 2) {
                z0 += p.b2[32 * half + 2 * i];
                z1 += p.b2[32 * half + 2 * i + 1];
            } else if constexpr (LAYER == 3) {
                z0 += p.b2b[32 * half + 2 * i];
                z1 += p.b2b[32 * half + 2 * i + 1];
            }
            h[16 * half + i] = pack_half2(hardgelu(z0), hardgelu(z1));
        }
    }
}

template <class P, int HM>
struct DecodeSmem {
    static constexpr uint32_t W1_BYTES = P::K1_ATOMS * 64 * 128;
    static constexpr uint32_t W2_BYTES = 64 * 128;
    static constexpr uint32_t W3_BYTES = 16 * 128;
    static constexpr uint32_t WIMG = W1_BYTES + HM * W2_BYTES + W3_BYTES;
    static constexpr uint32_t ABUF = P::K1_ATOMS * 128 * 128;
    static constexpr uint32_t BYTES = 1024 /*align slack*/ + WIMG + NWG * ABUF + 128 /*pe*/ + 64 /*bars*/ + 16;
};

template <class P, int HM>
__global__ void __launch_bounds__(NWG * 128, 1) decode_kernel(const __grid_constant__ DecodeParams p) {
    using S = DecodeSmem<P, HM>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* s_w = smem;
    uint8_t* s_a = smem + S::WIMG;
    uint32_t* s_pe = reinterpret_cast<uint32_t*>(s_a + NWG * S::ABUF);
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_pe + 32);
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_bar + NWG);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wg = warp >> 2, q = warp & 3, row = q * 32 + lane;

    for (uint32_t i = tid; i < S::WIMG / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(s_w)[i] = p.wimg[i];
    if (tid < 32) s_pe[tid] = (&p.pe_words[0][0])[tid];
    if (tid == 0) {
        for (int i = 0; i < NWG; ++i) mbar_init(&s_bar[i], 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(s_tmem, 512);
        tmem_relinquish();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    const uint32_t tmem = *s_tmem;
    const uint32_t t_d = tmem + (uint32_t)wg * 128u;             // this warpgroup's columns
    const uint32_t t_row = t_d + ((uint32_t)(q * 32) << 16);      // this warp's lane quarter
    const uint32_t a_tile = smem_u32(s_a + wg * S::ABUF);
    const uint32_t w1 = smem_u32(s_w), w2 = w1 + S::W1_BYTES, w3 = w2 + HM * S::W2_BYTES;
    const bool issuer = (q == 0) && (lane == 0);
    constexpr uint32_t ID64 = idesc_f16(128, 64), ID16 = idesc_f16(128, 16);
    uint32_t phase = 0;

    const int64_t ntiles = p.mode == 0 ? p.n_tiles : (p.nq + TILE_M - 1) / TILE_M;
    for (int64_t tile = (int64_t)blockIdx.x * NWG + wg; tile < ntiles; tile += (int64_t)gridDim.x * NWG) {
        // ---- resolve this thread's texel
        int m, x, y;
        bool valid, bad = false;
        uint16_t* dst;
        if (p.mode == 0) {
            int mi = 0;
            while (tile >= p.tile_start[mi + 1]) ++mi;
            m = p.mip_first + mi;
            const int64_t local = (tile - p.tile_start[mi]) * TILE_M + row;
            const int lw = p.M - 1 - m;  // log2(w_m)
            valid = local < ((int64_t)1 << (2 * lw));
            x = (int)(local & ((1 << lw) - 1));
            y = (int)(local >> lw);
            if (!valid) x = y = 0;
            dst = p.out + p.out_off[mi] + (int64_t)y * p.row_stride[mi] + (int64_t)x * p.c;
        } else {
            const int64_t qi = tile * TILE_M + row;
            valid = qi < p.nq;
            m = 0;
            x = y = 0;
            if (valid) {
                const uint2 qq = __ldg(reinterpret_cast<const uint2*>(p.q) + qi);
                x = (int)(qq.x & 0xFFFFu);
                y = (int)(qq.x >> 16);
                m = (int)(qq.y & 0xFFu);
                if (m >= p.M || x >= (p.W >> m) || y >= (p.W >> m)) {
                    bad = true;
                    m = p.M - 1;
                    x = y = 0;
                }
            }
            dst = p.out + qi * p.c;
        }
        // ---- a1-a4: assemble X into the swizzled A tile
        {
            uint32_t xw[P::K1W];
            assemble_row<P>(p, s_pe, m, x, y, xw, nullptr);
            store_row<P::K1W>(a_tile, row, xw);
        }
        fence_proxy_async_smem();
        tc_fence_before();
        named_bar_sync(1 + wg, 128);
        // ---- a5: D = X * W1^T (b1 folded through the constant-1 column)
        if (issuer) {
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < P::K1 / 16; ++k) {
                const uint64_t ad = umma_desc_k_sw128(a_tile + (k >> 2) * (128 * 128) + (k & 3) * 32);
                const uint64_t bd = umma_desc_k_sw128(w1 + (k >> 2) * (64 * 128) + (k & 3) * 32);
                mma_f16_ss(t_d, ad, bd, ID64, k > 0);
            }
            mma_commit(&s_bar[wg]);
        }
        mbar_wait(&s_bar[wg], phase);
        phase ^= 1;
        tc_fence_after();
        // ---- hidden layers
#pragma unroll
        for (int layer = 1; layer <= HM; ++layer) {
            uint32_t h[32];
            if (layer == 1)
                epilogue_hidden<1>(p, t_row, h);
            else
                epilogue_hidden<2>(p, t_row, h);
            store_row<32>(a_tile, row, h);
            fence_proxy_async_smem();
            tc_fence_before();
            named_bar_sync(1 + wg, 128);
            if (issuer) {
                tc_fence_after();
                const uint32_t wl = w2 + (layer - 1) * S::W2_BYTES;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    mma_f16_ss(t_d, umma_desc_k_sw128(a_tile + k * 32), umma_desc_k_sw128(wl + k * 32), ID64, k > 0);
                mma_commit(&s_bar[wg]);
            }
            mbar_wait(&s_bar[wg], phase);
            phase ^= 1;
            tc_fence_after();
        }
        {
            uint32_t h[32];
            if (HM == 1)
                epilogue_hidden<2>(p, t_row, h);
            else
                epilogue_hidden<3>(p, t_row, h);
            store_row<32>(a_tile, row, h);
        }
        fence_proxy_async_smem();
        tc_fence_before();
        named_bar_sync(1 + wg, 128);
        // ---- a7: Y = H * W3^T (N = 16) into columns [64, 80)
        if (issuer) {
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < 4; ++k)
                mma_f16_ss(t_d + 64, umma_desc_k_sw128(a_tile + k * 32), umma_desc_k_sw128(w3 + k * 32), ID16, k > 0);
            mma_commit(&s_bar[wg]);
        }
        mbar_wait(&s_bar[wg], phase);
        phase ^= 1;
        tc_fence_after();
        {
            uint32_t r[16];
            tmem_ld16(t_row + 64, r);
            tmem_wait_ld();
            if (valid) {
#pragma unroll
                for (int ch = 0; ch < 16; ++ch) {
                    if (ch < p.c) {
                        const float v = __saturatef(__uint_as_float(r[ch]) + p.b3[ch]);  // R13
                        dst[ch] = bad ? (uint16_t)0x7E00u : __half_as_ushort(__float2half_rn(v));
                    }
                }
                if (bad && p.status) atomicOr(p.status, (int)NTC_ERR_OUT_OF_RANGE);
            }
        }
        tc_fence_before();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

// Tests only: the same addressing + assembly, written to global memory.
template <class P>
__global__ void debug_assemble_kernel(const __grid_constant__ DecodeParams p) {
    __shared__ __align__(16) uint32_t s_pe[32];
    if (threadIdx.x < 32) s_pe[threadIdx.x] = (&p.pe_words[0][0])[threadIdx.x];
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.nq) return;
    const uint2 qq = reinterpret_cast<const uint2*>(p.q)[i];
    int x = (int)(qq.x & 0xFFFFu), y = (int)(qq.x >> 16), m = (int)(qq.y & 0xFFu);
    if (m >= p.M || x >= (p.W >> m) || y >= (p.W >> m)) {
        m = p.M - 1;
        x = y = 0;
    }
    uint32_t w[P::K1W];
    assemble_row<P>(p, s_pe, m, x, y, w, p.dbg_addr + i * 17);
    uint16_t* X = p.dbg_X + i * P::D;
    for (int k = 0; k < P::D; ++k) X[k] = (uint16_t)(w[k >> 1] >> (16 * (k & 1)));
}

// ------------------------------------------------------------------ launchers
template <class P, int HM>
static cudaError_t launch_decode_t(const DecodeParams& p, int grid, cudaStream_t s) {
    using S = DecodeSmem<P, HM>;
    auto* k = decode_kernel<P, HM>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, S::BYTES);
    if (e != cudaSuccess) return e;
    k<<<grid, NWG * 128, S::BYTES, s>>>(p);
    return cudaGetLastError();
}

template <class P>
static cudaError_t launch_debug_t(const DecodeParams& p, cudaStream_t s) {
    const int64_t blocks = (p.nq + 127) / 128;
    debug_assemble_kernel<P><<<(unsigned)blocks, 128, 0, s>>>(p);
    return cudaGetLastError();
}

using NTC02 = Prof<8, 2, 12, 4>;
using NTC05 = Prof<12, 4, 20, 4>;
using NTC10 = Prof<12, 2, 10, 4>;
using NTC225 = Prof<16, 4, 12, 4>;

int profile_id(const ntc_desc* d) {
    if (d->c0 == 8 && d->b0 == 2 && d->c1 == 12 && d->b1 == 4) return 0;
    if (d->c0 == 12 && d->b0 == 4 && d->c1 == 20 && d->b1 == 4) return 1;
    if (d->c0 == 12 && d->b0 == 2 && d->c1 == 10 && d->b1 == 4) return 2;
    if (d->c0 == 16 && d->b0 == 4 && d->c1 == 12 && d->b1 == 4) return 3;
    return -1;
}

uint32_t decode_wimg_bytes(int pid, int hm) {
    switch (pid) {
        case 0: return hm == 1 ? DecodeSmem<NTC02, 1>::WIMG : DecodeSmem<NTC02, 2>::WIMG;
        case 1: return hm == 1 ? DecodeSmem<NTC05, 1>::WIMG : DecodeSmem<NTC05, 2>::WIMG;
        case 2: return hm == 1 ? DecodeSmem<NTC10, 1>::WIMG : DecodeSmem<NTC10, 2>::WIMG;
        default: return hm == 1 ? DecodeSmem<NTC225, 1>::WIMG : DecodeSmem<NTC225, 2>::WIMG;
    }
}

int decode_k1(int pid) {
    switch (pid) {
        case 0: return NTC02::K1;
        case 1: return NTC05::K1;
        case 2: return NTC10::K1;
        default: return NTC225::K1;
    }
}

cudaError_t launch_decode(int pid, int hm, const DecodeParams& p, int grid, cudaStream_t s) {
    switch (pid * 2 + (hm - 1)) {
        case 0: return launch_decode_t<NTC02, 1>(p, grid, s);
        case 1: return launch_decode_t<NTC02, 2>(p, grid, s);
        case 2: return launch_decode_t<NTC05, 1>(p, grid, s);
        case 3: return launch_decode_t<NTC05, 2>(p, grid, s);
        case 4: return launch_decode_t<NTC10, 1>(p, grid, s);
        case 5: return launch_decode_t<NTC10, 2>(p, grid, s);
        case 6: return launch_decode_t<NTC225, 1>(p, grid, s);
        default: return launch_decode_t<NTC225, 2>(p, grid, s);
    }
}

cudaError_t launch_debug_assemble(int pid, const DecodeParams& p, cudaStream_t s) {
    switch (pid) {
        case 0: return launch_debug_t<NTC02>(p, s);
        case 1: return launch_debug_t<NTC05>(p, s);
        case 2: return launch_debug_t<NTC10>(p, s);
        default: return launch_debug_t<NTC225>(p, s);
    }
}

}  // namespace ntc
