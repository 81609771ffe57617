// assemble.cuh -- per-texel addressing, latent fetch and fp16 input-row assembly shared by
// the decode kernels and the debug export (product code).
//
// X column order inside the GPU path: the G0 part is permuted so that two codes can be
// dequantised with one byte-permute + mask + HFMA2 (see g0_word_cols); the W1 image is
// permuted identically (the MLP is invariant under a joint permutation of X and W1's
// columns) and ntc_debug_assemble un-permutes to the canonical order of reading R4.
#pragma once
#include <cuda_fp16.h>

#include "common.cuh"
#include "ptx.cuh"

namespace ntc {

// ------------------------------------------------------------------ G0 column permutation
// word index wi in [0, 2*C0) of the G0 part, lane l in {0,1} -> canonical X column
// (tap * C0 + channel) of reading R4.
__host__ __device__ constexpr int g0_word_col(int C0, int B0, int wi, int l) {
    if (C0 == 8 && B0 == 2) {  // per tap: (k, k+4)
        return (wi / 4) * 8 + (wi % 4) + 4 * l;
    }
    if (C0 == 12 && B0 == 2) {  // per tap (k, k+4) from bytes 0/1; byte 2 paired across taps
        if (wi < 16) return (wi / 4) * 12 + (wi % 4) + 4 * l;
        const int j = wi - 16, pi = j / 4, k = j % 4;
        return (2 * pi + l) * 12 + 8 + k;
    }
    if (C0 == 12 && B0 == 4) {  // per tap: (q, q+4) q<4 ; (8+q, 10+q) q<2
        const int t = wi / 6, k = wi % 6;
        return t * 12 + (k < 4 ? k + 4 * l : 8 + (k - 4) + 2 * l);
    }
    if (C0 == 16 && B0 == 4) {  // per tap: (q, q+4) ; (8+q, 12+q)
        const int t = wi / 8, k = wi % 8;
        return t * 16 + (k < 4 ? k + 4 * l : 8 + (k - 4) + 4 * l);
    }
    return -1;
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
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(base) + idx);
        c.w[0] = v.x;
        c.w[1] = v.y;
    } else {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(base) + idx);
        c.w[0] = v.x;
        c.w[1] = v.y;
        c.w[2] = v.z;
        c.w[3] = v.w;
    }
    return c;
}

// dequantise the two codes held in bits [SH,SH+B) and [16+SH,16+SH+B) of `lanes` (already
// masked, SH + B <= 10): half(0x6400 | code << SH) = 1024 + code 2^SH; one HFMA2 with the
// power-of-2 scale Q / 2^SH gives (code - N/2 + 1) / N exactly (R10): the
// product is exact and the result is representable, so the single rounding is exact.
template <int B, int SH = 0, bool MAGIC_SET = false>
__device__ __forceinline__ uint32_t dequant2(uint32_t lanes) {
    static_assert(SH + B <= 10, "code bits must stay inside the fp16 mantissa");
    constexpr float Q = 1.0f / (float)(1 << B);
    constexpr float OFF = (float)((1 << B) / 2 - 1);
    constexpr float SC = Q / (float)(1 << SH);
    // MAGIC_SET: the caller already ORed in 0x64006400 (one fused lop3 with its mask)
    const uint32_t v = MAGIC_SET ? lanes : lanes | 0x64006400u;
    __half2 r = __hfma2(*reinterpret_cast<const __half2*>(&v), __float2half2_rn(SC),
                        __float2half2_rn(-(1024.0f / (float)(1 << SH) + OFF) * Q));
    return *reinterpret_cast<uint32_t*>(&r);
}

// (y & mask) | 0x64006400 as ONE lop3 (ptxas splits it into two LOP3s when both constants are
// immediates); dequant2<..., true> then skips its own OR
__device__ __forceinline__ uint32_t mask_or_magic(uint32_t y, uint32_t mask) {
    uint32_t v;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(v) : "r"(y), "r"(mask), "r"(0x64006400u));
    return v;
}

// 4-bit codes: split a 32-bit word of `nch` channels into lane pairs (bits 0-3 | 16-19)
// (MAGIC: each lane pair already ORed with the fp16 magic 0x6400 by the same lop3)
template <int NCH, bool MAGIC = false>
__device__ __forceinline__ void nib_lanes(uint32_t w, uint32_t* out) {
    auto m = [](uint32_t v) { return MAGIC ? mask_or_magic(v, 0x000F000Fu) : v & 0x000F000Fu; };
    if constexpr (NCH == 8) {
#pragma unroll
        for (int q = 0; q < 4; ++q) out[q] = m(w >> (4 * q));  // (q, q+4)
    } else if constexpr (NCH == 4) {
        const uint32_t y = __byte_perm(w, 0u, 0x4140);       // [b0, 0, b1, 0]
        out[0] = m(y);                                        // (0, 2)
        out[1] = m(y >> 4);                                   // (1, 3)
    } else {
        const uint32_t y = w | (w << 12);
        out[0] = m(y);                                        // (0, 1)
    }
}

// G1 variant: lane pairs with the code at bit 0 or bit 4 of each 16-bit lane (scale 1 or 16;
// G1 sums stay below 2^16 either way: 16 * 15 * 256 = 61440), which saves the shifts
template <int NCH>
__device__ __forceinline__ void nib_lanes_g1(uint32_t w, uint32_t* out) {
    if constexpr (NCH == 8) {
        const uint32_t h = w >> 8;
        out[0] = w & 0x000F000Fu;  // (0, 4) x1
        out[1] = w & 0x00F000F0u;  // (1, 5) x16
        out[2] = h & 0x000F000Fu;  // (2, 6) x1
        out[3] = h & 0x00F000F0u;  // (3, 7) x16
    } else if constexpr (NCH == 4) {
        const uint32_t y = __byte_perm(w, 0u, 0x4140);  // [b0, 0, b1, 0]
        out[0] = y & 0x000F000Fu;                        // (0, 2) x1
        out[1] = y & 0x00F000F0u;                        // (1, 3) x16
    } else {
        const uint32_t y = w | (w << 12);
        out[0] = y & 0x000F000Fu;                        // (0, 1) x1
    }
}

// ------------------------------------------------------------------ fetch (a1 + loads)
template <class P>
struct Fetch {
    Cell<P::CELL0> g0[4];
    Cell<P::CELL1> g1[4];
    // packed (one register, it lives across a whole tile): x mod 8 [0,3), y mod 8 [3,6),
    // mip [6,10), G1 fractional offsets ax [10,15) and ay [15,20) in 1/16 (exact), then the
    // decode kernel's row flags: valid (bit 20), bad query (bit 21)
    uint32_t info;
    uint16_t* dst;   // output row of this texel
};
__device__ __forceinline__ int info_px(uint32_t i) { return (int)(i & 7u); }
__device__ __forceinline__ int info_py(uint32_t i) { return (int)((i >> 3) & 7u); }
__device__ __forceinline__ int info_m(uint32_t i) { return (int)((i >> 6) & 15u); }
__device__ __forceinline__ uint32_t info_ax(uint32_t i) { return (i >> 10) & 31u; }
__device__ __forceinline__ uint32_t info_ay(uint32_t i) { return (i >> 15) & 31u; }

// R1/R2/R3: u = (x + 1/2) r / w_m - 1/2 with clamp-to-edge taps (i, j), (i+1, j), (i, j+1),
// (i+1, j+1).  All sizes are powers of two, so in integers: num = (2x + 1) r - w_m,
// i = floor(num / 2 w_m) (arithmetic shift), frac = (num mod 2 w_m) / 2 w_m.  The G1
// fractional offsets are multiples of 1/16 (r1 / w_m >= 1/8 for every compiled profile),
// so the bilinear weights are exact multiples of 1/256.
template <class P>
__device__ __forceinline__ void fetch_texel(const DecodeParams& p, const uint8_t* grids, int m, int x, int y,
                                            Fetch<P>& f, int32_t* dbg_addr) {
    const int j = p.level_of[m];
    const LevelGeom g = p.lv[j];
    const int lw = p.M - 1 - m;  // log2(w_m)
    const int xs = 2 * x + 1, ys = 2 * y + 1;
    int tx0[2], ty0[2], tx1[2], ty1[2];
    {
        const int nx = (xs << g.lr0) - (1 << lw), ny = (ys << g.lr0) - (1 << lw);
        const int i = nx >> (lw + 1), k = ny >> (lw + 1);
        tx0[0] = max(i, 0);
        tx0[1] = min(i + 1, g.r0 - 1);
        ty0[0] = max(k, 0);
        ty0[1] = min(k + 1, g.r0 - 1);
    }
    {
        const int nx = (xs << g.lr1) - (1 << lw), ny = (ys << g.lr1) - (1 << lw);
        const int i = nx >> (lw + 1), k = ny >> (lw + 1);
        const int mask = (2 << lw) - 1;
        const uint32_t ax = (uint32_t)(((nx & mask) << 4) >> (lw + 1));
        const uint32_t ay = (uint32_t)(((ny & mask) << 4) >> (lw + 1));
        f.info = (uint32_t)(x & 7) | ((uint32_t)(y & 7) << 3) | ((uint32_t)m << 6) | (ax << 10) | (ay << 15);
        tx1[0] = max(i, 0);
        tx1[1] = min(i + 1, g.r1 - 1);
        ty1[0] = max(k, 0);
        ty1[1] = min(k + 1, g.r1 - 1);
    }
    const uint8_t* g0 = grids + g.off0;
    const uint8_t* g1 = grids + g.off1;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        f.g0[t] = load_cell<P::CELL0>(g0, (uint32_t)(ty0[t >> 1] * g.r0 + tx0[t & 1]));
        f.g1[t] = load_cell<P::CELL1>(g1, (uint32_t)(ty1[t >> 1] * g.r1 + tx1[t & 1]));
    }
    if (dbg_addr) {
        dbg_addr[0] = j;
        for (int t = 0; t < 4; ++t) {
            dbg_addr[1 + 2 * t] = tx0[t & 1];
            dbg_addr[2 + 2 * t] = ty0[t >> 1];
            dbg_addr[9 + 2 * t] = tx1[t & 1];
            dbg_addr[10 + 2 * t] = ty1[t >> 1];
        }
    }
}

// ------------------------------------------------------------------ assembly pieces
// G0 of NTC 0.2 (C0 = 8, B0 = 2): 16 words from the four 16-bit tap cells
__device__ __forceinline__ void g0_words_c8b2(const uint32_t (&cell)[4], uint32_t (&w)[16]) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const uint32_t y = __byte_perm(cell[t], 0u, 0x4140);
        w[4 * t + 0] = dequant2<2, 0, true>(mask_or_magic(y, 0x00030003u));
        w[4 * t + 1] = dequant2<2, 2, true>(mask_or_magic(y, 0x000C000Cu));
        w[4 * t + 2] = dequant2<2, 4, true>(mask_or_magic(y, 0x00300030u));
        w[4 * t + 3] = dequant2<2, 6, true>(mask_or_magic(y, 0x00C000C0u));
    }
}

// G1: bilinear as integer multiply-adds on two 16-bit lanes:
// S = sum_t wt_t * code_t (< 2^16), value = (S - 256 (N/2-1)) / (256 N), exact in fp32,
// rounded once to fp16.  cell[t][wd]: 32-bit word wd of tap t's packed cell.
template <class P, int NWD>
__device__ __forceinline__ void g1_words(const uint32_t (&cell)[4][NWD], const uint32_t (&wt)[4],
                                         uint32_t (&out)[P::C1 / 2]) {
    static_assert(P::B1 == 4, "G1 path assumes 4-bit codes (all Table 2 profiles)");
    constexpr int NL = P::C1 / 2;
    uint32_t S[NL];
    float v[P::C1];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        uint32_t l[NL];
        int cb[NL];  // first channel of each lane pair, second = cb + step
        int st[NL];
        float sc[NL];  // lane scale: the code sits at bit 0 (1) or bit 4 (16) of its lane
        int n = 0;
#pragma unroll
        for (int wd = 0; wd * 8 < P::C1; ++wd) {
            const int nch = P::C1 - wd * 8 >= 8 ? 8 : P::C1 - wd * 8;
            if (nch == 8) {
                nib_lanes_g1<8>(cell[t][wd], l + n);
#pragma unroll
                for (int q = 0; q < 4; ++q) { cb[n + q] = wd * 8 + q; st[n + q] = 4; sc[n + q] = (q & 1) ? 16.0f : 1.0f; }
                n += 4;
            } else if (nch == 4) {
                nib_lanes_g1<4>(cell[t][wd], l + n);
#pragma unroll
                for (int q = 0; q < 2; ++q) { cb[n + q] = wd * 8 + q; st[n + q] = 2; sc[n + q] = q ? 16.0f : 1.0f; }
                n += 2;
            } else {
                nib_lanes_g1<2>(cell[t][wd], l + n);
                cb[n] = wd * 8;
                st[n] = 1;
                sc[n] = 1.0f;
                n += 1;
            }
        }
#pragma unroll
        for (int i = 0; i < NL; ++i) S[i] = t == 0 ? l[i] * wt[0] : S[i] + l[i] * wt[t];
        if (t == 3) {
            // value = (S / scale - 256 (N/2 - 1)) / (256 N) with S read as 2^23 + S (exact)
            constexpr float SC = 1.0f / (256.0f * 16.0f);
#pragma unroll
            for (int i = 0; i < NL; ++i) {
                const float sci = SC / sc[i], bi = -(8388608.0f / sc[i] + 256.0f * 7.0f) * SC;
                v[cb[i]] = fmaf(__uint_as_float(__byte_perm(S[i], 0x4B000000u, 0x7610)), sci, bi);
                v[cb[i] + st[i]] = fmaf(__uint_as_float(__byte_perm(S[i], 0x4B000000u, 0x7632)), sci, bi);
            }
        }
    }
#pragma unroll
    for (int k = 0; k < P::C1 / 2; ++k) out[k] = pack_half2(v[2 * k], v[2 * k + 1]);
}

// PE from the per-axis table, then LOD + bias one: 7 words
__device__ __forceinline__ void pe_lod_words(const DecodeParams& p, const uint32_t* s_pe, int m, int x, int y,
                                             uint32_t (&w)[7]) {
    const uint4 px = *reinterpret_cast<const uint4*>(s_pe + 4 * (x & 7));
    const uint4 py = *reinterpret_cast<const uint4*>(s_pe + 4 * (y & 7));
    w[0] = px.x;
    w[1] = px.y;
    w[2] = px.z;
    w[3] = py.x;
    w[4] = py.y;
    w[5] = py.z;
    w[6] = p.lod_word[m];
}

// ------------------------------------------------------------------ assembly (a2-a4)
// X = [G0 taps (permuted pairs) | bilinear G1 | PE_x(6) | PE_y(6) | LOD | 1 | 0 ...] as
// K1W half2 words; the trailing 1 multiplies the b1 column of the W1 image.
template <class P>
__device__ __forceinline__ void assemble_words(const DecodeParams& p, const uint32_t* s_pe, const Fetch<P>& f,
                                               uint32_t (&w)[P::K1W]) {
    // ---- G0: four unfiltered taps (learned interpolation)
    if constexpr (P::C0 == 8 && P::B0 == 2) {
        const uint32_t cell[4] = {f.g0[0].w[0], f.g0[1].w[0], f.g0[2].w[0], f.g0[3].w[0]};
        uint32_t g[16];
        g0_words_c8b2(cell, g);
#pragma unroll
        for (int i = 0; i < 16; ++i) w[i] = g[i];
    } else if constexpr (P::C0 == 12 && P::B0 == 2) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const uint32_t y = __byte_perm(f.g0[t].w[0], 0u, 0x4140);
#pragma unroll
            for (int k = 0; k < 4; ++k) w[4 * t + k] = dequant2<2, 0, true>(mask_or_magic(y >> (2 * k), 0x00030003u));
        }
#pragma unroll
        for (int pi = 0; pi < 2; ++pi) {
            const uint32_t y = __byte_perm(f.g0[2 * pi].w[0], f.g0[2 * pi + 1].w[0], 0x7672);
#pragma unroll
            for (int k = 0; k < 4; ++k)
                w[16 + 4 * pi + k] = dequant2<2, 0, true>(mask_or_magic(y >> (2 * k), 0x00030003u));
        }
    } else if constexpr (P::C0 == 12 && P::B0 == 4) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            uint32_t l[6];
            nib_lanes<8, true>(f.g0[t].w[0], l);
            nib_lanes<4, true>(f.g0[t].w[1], l + 4);
#pragma unroll
            for (int k = 0; k < 6; ++k) w[6 * t + k] = dequant2<4, 0, true>(l[k]);
        }
    } else {
        static_assert(P::C0 == 16 && P::B0 == 4, "unsupported G0 profile");
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            uint32_t l[8];
            nib_lanes<8, true>(f.g0[t].w[0], l);
            nib_lanes<8, true>(f.g0[t].w[1], l + 4);
#pragma unroll
            for (int k = 0; k < 8; ++k) w[8 * t + k] = dequant2<4, 0, true>(l[k]);
        }
    }
    // ---- G1 bilinear, PE, LOD
    {
        constexpr int NWD = P::CELL1 >= 4 ? P::CELL1 / 4 : 1;
        uint32_t cell[4][NWD];
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int wd = 0; wd < NWD; ++wd) cell[t][wd] = f.g1[t].w[wd];
        uint32_t g[P::C1 / 2];
        const uint32_t ax = info_ax(f.info), ay = info_ay(f.info);
        const uint32_t wt[4] = {(16u - ax) * (16u - ay), ax * (16u - ay), (16u - ax) * ay, ax * ay};
        g1_words<P, NWD>(cell, wt, g);
#pragma unroll
        for (int k = 0; k < P::C1 / 2; ++k) w[2 * P::C0 + k] = g[k];
    }
    constexpr int PEW = (4 * P::C0 + P::C1) / 2;
    {
        uint32_t pw[7];
        pe_lod_words(p, s_pe, info_m(f.info), info_px(f.info), info_py(f.info), pw);
#pragma unroll
        for (int k = 0; k < 7; ++k) w[PEW + k] = pw[k];
    }
#pragma unroll
    for (int k = PEW + 7; k < P::K1W; ++k) w[k] = 0u;
}

// canonical (R4) column of GPU X column `col`
template <class P>
__host__ __device__ constexpr int canonical_col(int col) {
    return col < 4 * P::C0 ? g0_word_col(P::C0, P::B0, col / 2, col & 1) : col;
}

}  // namespace ntc
