// decode.cu -- per-texel NTC decode on sm_100a (tcgen05 + TMEM), product code.
//
// One persistent CTA per SM, 4 warpgroups (2 for profiles with K1 > 64).  Each warpgroup
// ping-pongs between two 128-texel tile contexts (TMEM lane r <-> texel r <-> thread r of
// the warpgroup), so the tensor core works on one context while the threads run the
// other's epilogue:
//   a1     every thread resolves its texel of the NEXT tile and issues its 8 latent-cell
//          loads, which stay in flight while the current tile runs through the MLP;
//   a2-a4  it assembles its fp16 input row X (G0 2x2 gather, G1 bilinear, PE, LOD, a
//          constant 1 for the folded bias b1) into a K-major, 128B-swizzled SMEM tile;
//   a5-a7  one elected thread issues tcgen05.mma per layer (M=128; N=64, 64, 16); the
//          biases of layers 2/3 enter as one extra K=16 MMA against a constant ones tile;
//          the epilogue is tcgen05.ld -> hardGELU (FFMA.SAT + packed FMUL2) -> fp16 ->
//          SMEM A operand of the next layer; the output is clamped to [0,1] and stored.
// The whole MLP weight set lives in SMEM for the CTA's lifetime (one copy per SM).
#include <cuda_fp16.h>

#include <type_traits>

#include "assemble.cuh"
#include "common.cuh"
#include "ptx.cuh"

namespace ntc {

// store NW half2 words of row `row` into the A tile of 128 rows: K columns [0, 64) in a
// K-major SW128 atom, the rest (K1 = 80 / 96) in a K-major SW32 / SW64 part right after it
template <int NW>
__device__ __forceinline__ void store_row(uint32_t tile, int row, const uint32_t* w) {
    constexpr int K2B = NW * 4 - 128;  // bytes per row of the second part (0, 32 or 64)
#pragma unroll
    for (int c = 0; c < NW / 4; ++c) {
        uint32_t addr;
        if (c < 8) {
            addr = tile + (uint32_t)row * 128u + ((uint32_t)(c ^ (row & 7)) << 4);
        } else {
            const uint32_t j = (uint32_t)(c - 8);
            const uint32_t sw = K2B == 32 ? ((row >> 2) & 1) : ((row >> 1) & 3);
            addr = tile + 128u * 128u + (uint32_t)row * K2B + ((j ^ sw) << 4);
        }
        sts128(addr, w[4 * c + 0], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
    }
}

// hardGELU of a column pair: z * sat(z/3 + 1/2), packed fp32 multiply
__device__ __forceinline__ uint32_t hardgelu2(uint32_t a, uint32_t b) {
    const float2 z = make_float2(__uint_as_float(a), __uint_as_float(b));
    const float2 t = make_float2(__saturatef(fmaf(z.x, 1.0f / 3.0f, 0.5f)), __saturatef(fmaf(z.y, 1.0f / 3.0f, 0.5f)));
    const float2 h = __fmul2_rn(z, t);
    return pack_half2(h.x, h.y);
}

// exact GELU of a column pair: z Phi(z) = z/2 (1 + erf(z / sqrt 2)) (f4 variant)
__device__ __forceinline__ uint32_t gelu2(uint32_t a, uint32_t b) {
    const float za = __uint_as_float(a), zb = __uint_as_float(b);
    return pack_half2(0.5f * za * (1.0f + erff(za * 0.70710678118654752f)),
                      0.5f * zb * (1.0f + erff(zb * 0.70710678118654752f)));
}

template <int ACT>
__device__ __forceinline__ uint32_t act2(uint32_t a, uint32_t b) {
    if constexpr (ACT == 0)
        return hardgelu2(a, b);
    else
        return gelu2(a, b);
}

// TMEM accumulator columns [0, 64) of this thread's lane (bias already accumulated)
// -> hardGELU (or GELU) -> fp16 -> row `row` of the SW128 A tile, 32 columns at a time
template <int ACT, bool PIPE>
__device__ __forceinline__ void epilogue_hidden(uint32_t taddr, uint32_t tile, int row) {
    if constexpr (!PIPE) {  // two 32-column halves, each loaded then processed
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            uint32_t r[32];
            tmem_ld32(taddr + 32 * half, r);
            tmem_wait_ld();
            uint32_t h[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) h[i] = act2<ACT>(r[2 * i], r[2 * i + 1]);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int chunk = 4 * half + c;
                sts128(tile + (uint32_t)row * 128u + ((uint32_t)(chunk ^ (row & 7)) << 4), h[4 * c], h[4 * c + 1],
                       h[4 * c + 2], h[4 * c + 3]);
            }
        }
        return;
    }
    // PIPE: 16-column chunks, the next one's tcgen05.ld in flight while this one is processed
    // (and 16 fewer live registers, which removes the spills of the mip-tile instantiations)
    uint32_t r[2][16];
    tmem_ld16(taddr, r[0]);
    tmem_wait_ld_r16(r[0]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (q < 3) tmem_ld16(taddr + 16 * (q + 1), r[(q + 1) & 1]);
        uint32_t h[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) h[i] = act2<ACT>(r[q & 1][2 * i], r[q & 1][2 * i + 1]);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int chunk = 2 * q + c;
            sts128(tile + (uint32_t)row * 128u + ((uint32_t)(chunk ^ (row & 7)) << 4), h[4 * c], h[4 * c + 1],
                   h[4 * c + 2], h[4 * c + 3]);
        }
        if (q < 3) tmem_wait_ld_r16(r[(q + 1) & 1]);
    }
}

#ifndef DECODE_NWG
#define DECODE_NWG 4
#endif
// 1: mip-tile output staged in SMEM and written by one bulk TMA store per tile (K1 = 64
// profiles, whose SMEM has room for the 8 staging buffers); 0 (default): every thread stores
// its own row.  A/B on B200 (tools/ab_decode.py, 3 alternating runs): the bulk store path is
// 3% slower (4K chain c = 9: 29.05 vs 29.97 Gtexel/s; c = 16: 29.17 vs 30.23), so it stays off.
#ifndef DECODE_TMA_OUT
#define DECODE_TMA_OUT 0
#endif
// Where a context issues the latent loads of its next tile: 0 right after its MMA1 issue (end
// of phase 0); 1 at the start of its second hidden phase, before that phase's MMA wait -- the
// wait that otherwise has only the other context's first epilogue to hide behind (A/B: 1 is
// 3-5% slower, the loads then land too late for the next assembly; 0 kept).
// 1: the MMAs of the uniform-register instantiations are issued by the whole issuing warp
// through elect.sync (no per-MMA single-thread waterfall); 2: and each layer's MMAs + commit as
// one asm block; 0: by lane 0 of that warp.  A/B on the 4K chain (3 rounds): 0 -> 1: c = 9
// 29.85 -> 30.61 Gtexel/s; 1 -> 2: c = 9 30.44 -> 32.34, c = 16 30.08 -> 32.34
#ifndef DECODE_WARP_ISSUE
#define DECODE_WARP_ISSUE 2
#endif
// 1: a steady-state loop without the per-phase idle checks while every context holds a tile
// (A/B: neutral on the chain decode, -4% on random queries; off)
// 1: the c = 16 query instantiation also gets the uniform-register MMA issue (A/B: random
// queries 20.6 -> 20.2 Gtexel/s, off)
// 1: the lane quarter goes through a shuffle as well (uniform-register instantiations).  A/B, 3
// rounds: 4K chain c = 9 32.33 -> 33.65 Gtexel/s, c = 16 32.30 -> 33.95, NTC 0.5 / 1.0 / 2.25
// 23.1 / 28.7 / 25.5 -> 25.3 / 30.8 / 28.2; ptxas: 114 -> 96 registers, R2UR 50 -> 4
#ifndef DECODE_UNI_Q
#define DECODE_UNI_Q 1
#endif
#ifndef DECODE_UNI_QUERY
#define DECODE_UNI_QUERY 0
#endif
#ifndef DECODE_WARP_ALL
#define DECODE_WARP_ALL 0
#endif
#ifndef DECODE_STEADY
#define DECODE_STEADY 0
#endif
#ifndef DECODE_FETCH_AT
#define DECODE_FETCH_AT 0
#endif
template <class P, int HM>
struct DecodeSmem {
    // K1 > 64 (NTC 0.5 / 1.0 / 2.25): the K columns past 64 live in a K-major SW32 (K1 = 80)
    // or SW64 (K1 = 96) part of 32 / 64 B per row after the SW128 atom, for the X tiles and W1
    static constexpr int K2 = P::K1_ATOMS == 2 ? P::K1 - 64 : 0;
    static constexpr uint32_t K2B = 2 * K2;
    static_assert(K2 == 0 || K2 == 16 || K2 == 32, "second K part: 16 or 32 columns");
    // warpgroups per CTA x tile contexts per warpgroup: 8 contexts x 64 TMEM columns = 512
    // (4 contexts for the K1 > 64 profiles at depth 2, whose SMEM does not fit 8)
    static constexpr bool FULL = P::K1_ATOMS == 1 || HM == 1;
    static constexpr int NWG = FULL ? DECODE_NWG : 2;
    static constexpr int NC = FULL ? 8 / DECODE_NWG : 2;
    static constexpr uint32_t W1_BYTES = 64 * 128 + 64 * K2B;
    static constexpr uint32_t W2_BYTES = 64 * 128 + 64 * 32;  // SW128 weights + SW32 bias atom
    static constexpr uint32_t W3_BYTES = 2 * 16 * 128;
    static constexpr uint32_t WIMG = W1_BYTES + HM * W2_BYTES + W3_BYTES;
    static constexpr uint32_t ONES = 128 * 32;  // constant SW32 A tile (K = 16): column 0 = 1
    static constexpr uint32_t ABUF = 128 * 128 + 128 * K2B;  // one per tile context
    // output staging for the bulk TMA store (tiled mode): 128 rows x c halves per context
    static constexpr bool TMA_OUT = DECODE_TMA_OUT && P::K1_ATOMS == 1;
    static constexpr uint32_t STAGE = TMA_OUT ? 128 * 16 * 2 : 0;
    static constexpr uint32_t BYTES =
        1024 + WIMG + ONES + NWG * NC * (ABUF + STAGE) + 128 /*pe*/ + 128 /*bars*/ + 16;
    static_assert(W1_BYTES % 1024 == 0 && W2_BYTES % 1024 == 0 && ABUF % 1024 == 0, "SW128 atoms 1 KB aligned");
    static_assert(BYTES <= 232448, "decode SMEM layout exceeds 227 KB");
};

// The tile range a CTA is working through, with the material it belongs to (uniform).
struct Run {
    const uint8_t* grids;
    const float* b3;
    int ts0, seg0, cnt;  // multi: first tile, first perm slot and query count of the material
    const int32_t* perm;
};

// resolve the texel of row `row` of `tile`, its output address, and issue its latent loads
template <class P, bool MULTI, int CT = 0, bool TILED = false>
__device__ __forceinline__ void fetch_tile(const DecodeParams& p, const Run R, int tile, int row, Fetch<P>& f) {
    int m = 0, x = 0, y = 0;
    bool valid, bad = false;
    if (TILED || (!MULTI && p.mode == 0)) {
        int mi = 0;
        if (tile >= p.tile_start[1])  // most tiles belong to the first mip
            while (tile >= p.tile_start[mi + 1]) ++mi;
        m = p.mip_first + mi;
        const int local = (tile - p.tile_start[mi]) * TILE_M + row;
        const int lw = p.M - 1 - m;  // log2(w_m)
        valid = local < (1 << (2 * lw));
        if (valid) {
            x = local & ((1 << lw) - 1);
            y = local >> lw;
        }
        if (tile < p.lin_tiles)  // uniform: the output row is texel tile * 128 + row of `out`
            f.dst = p.out + (int64_t)(tile * TILE_M + row) * (CT ? CT : p.c);
        else
            f.dst = p.out + (p.out_off[mi] + (int64_t)y * p.row_stride[mi] + x * (CT ? CT : p.c));
    } else {
        int64_t qi;
        if (MULTI) {
            const int local = (tile - R.ts0) * TILE_M + row;
            valid = local < R.cnt;
            qi = valid ? (int64_t)__ldg(R.perm + R.seg0 + local) : 0;
        } else {
            qi = (int64_t)tile * TILE_M + row;
            valid = qi < p.nq;
        }
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
        f.dst = p.out + qi * (CT ? CT : p.c);
    }
    fetch_texel<P>(p, MULTI ? R.grids : p.grids, m, x, y, f, nullptr);
    f.info |= ((uint32_t)valid << 20) | ((uint32_t)bad << 21);
}

// a7 store of one texel's c fp16 channels (o = 8 packed pairs).  c is uniform, so the
// branches below are uniform: even c with a 4-byte-aligned output -> b32 pairs (16-byte
// vectors for the compiled c = 16), otherwise b16 stores.
// pair (uniform per tile, odd c): rows 2i and 2i+1 are one 4-byte-aligned run of 2c halves;
// the even row's lane writes its (c+1)/2 words, the last one completed with the odd row's
// first channel (one shuffle), and the odd row's lane writes the remaining (c-1)/2 words.
template <int CT, bool TILED>
__device__ __forceinline__ void store_output(const DecodeParams& p, uint16_t* dst, bool valid, bool bad, bool pair,
                                             int row, const uint32_t (&o)[8]) {
    uint32_t v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = o[k];
    if (!TILED && p.mode != 0) {  // queries: NaN row for a bad one (uniform branch)
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = bad ? 0x7E007E00u : v[k];
        if (bad && p.status) atomicOr(p.status, (int)NTC_ERR_OUT_OF_RANGE);
    }
    const int c = CT ? CT : p.c;
    if (pair) {
        const uint32_t partner = __shfl_xor_sync(0xffffffffu, v[0], 1);
        const bool odd = row & 1;
        const uint32_t sel = odd ? 0x5432u : 0x3210u;
        uint32_t* d32 = reinterpret_cast<uint32_t*>(dst + (odd ? 1 : 0));
        const int nw = (c - 1) >> 1;
#pragma unroll
        for (int k = 0; k < 7; ++k)
            if (k < nw) d32[k] = __byte_perm(v[k], v[k + 1], sel);
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (k == nw && !odd) d32[k] = __byte_perm(v[k], partner, 0x5410);
        return;
    }
    if (!valid) return;
    if constexpr (CT > 0 && CT % 8 == 0) {  // 16-byte rows: vector stores when aligned
        if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
#pragma unroll
            for (int k = 0; k < CT / 8; ++k)
                reinterpret_cast<uint4*>(dst)[k] = make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
            return;
        }
    }
    if ((c & 1) == 0 && (reinterpret_cast<uintptr_t>(dst) & 3u) == 0) {
        uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (2 * k < c) d32[k] = v[k];
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (2 * k < c) dst[2 * k] = (uint16_t)(v[k] & 0xFFFFu);
            if (2 * k + 1 < c) dst[2 * k + 1] = (uint16_t)(v[k] >> 16);
        }
    }
}

// Per-warpgroup ping-pong over two tile contexts: while the tensor core runs one
// context's layer, the warpgroup's threads run the other context's epilogue.
template <class P>
struct Ctx {
    int tile;           // current tile of this context (>= ntiles: idle)
    Fetch<P> nxt;       // prefetched latents of the context's next tile
    uint16_t* dst;      // current texel's output row
    uint32_t flags;     // bit 0 valid, bit 1 bad query
    uint32_t phase;
    uint32_t abuf, tcol;
    uint64_t* bar;
    int id;             // context index (named barrier selector)
    int iq;             // warp (lane quarter) that issues this context's MMAs
    uint64_t adesc;     // SW128 K-major descriptor of abuf
    uint32_t stage;     // SMEM output staging (bulk TMA store)
    int ptile;          // tile whose staged output awaits its bulk store (-1: none)
};

// CT: the channel count as a compile-time constant (0: the runtime p.c), for the output path;
// TILED: compiled for mode 0 (tiles over mips) only
template <class P, int HM, bool MULTI, int ACT, int CT = 0, bool TILED = false>
__device__ __forceinline__ void decode_body(const DecodeParams& p, const MultiTable* mt) {
    using S = DecodeSmem<P, HM>;
    constexpr int NW = S::NWG, NC = S::NC;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* s_w = smem;
    uint8_t* s_ones = smem + S::WIMG;
    uint8_t* s_a = s_ones + S::ONES;
    uint8_t* s_stage = s_a + NW * NC * S::ABUF;
    uint32_t* s_pe = reinterpret_cast<uint32_t*>(s_stage + NW * NC * S::STAGE);
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_pe + 32);
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_bar + NC * NW);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // TILED instantiation: wg and the TMEM base go through a shuffle, which makes them provably
    // warp-uniform: the MMA-issuing thread then keeps descriptors, TMEM columns and mbarrier
    // addresses in uniform registers (no R2UR waterfall around each tcgen05.mma).  Measured
    // +2.7% on the headline chain decode; the query/multi instantiations ran slower with it
    // (more spills), so they keep the plain values.
    // uniform-register MMA issue (shuffled wg / TMEM base) and pipelined TMEM reads: mip
    // tiles and the compiled multi-material kernel; A/B-measured slower for the query kernel
    constexpr bool UNI = TILED || (MULTI && CT != 0) || (DECODE_UNI_QUERY && CT != 0);
    constexpr bool TMA = TILED && S::TMA_OUT;  // mip tiles: staged output, one bulk store per tile
    // (the lane quarter too, so the issuing-warp test `q == C.iq` is provably warp-uniform and the
    // elect.sync blocks need no divergence check)
    const int wg = UNI ? __shfl_sync(0xffffffffu, warp >> 2, 0) : warp >> 2;
    const int q = (UNI && DECODE_UNI_Q) ? __shfl_sync(0xffffffffu, warp & 3, 0) : warp & 3, row = q * 32 + lane;

    if (!MULTI)
        for (uint32_t i = tid; i < S::WIMG / 16; i += blockDim.x) reinterpret_cast<uint4*>(s_w)[i] = p.wimg[i];
    for (uint32_t i = tid; i < S::ONES / 16; i += blockDim.x) {
        const uint32_t r = i >> 1, chunk = i & 1;     // 16-byte chunk `chunk` of SW32 row r
        const bool one = chunk == ((r >> 2) & 1);     // logical chunk 0 lands at physical (r>>2)&1
        reinterpret_cast<uint4*>(s_ones)[i] = make_uint4(one ? 0x3C00u : 0u, 0u, 0u, 0u);
    }
    if (tid < 32) s_pe[tid] = (&p.pe_words[0][0])[tid];
    if (tid == 0) {
        for (int i = 0; i < NC * NW; ++i) mbar_init(&s_bar[i], 1);
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

    const uint32_t tmem = UNI ? __shfl_sync(0xffffffffu, *s_tmem, 0) : *s_tmem;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;   // this warp's TMEM lane quarter
    const uint32_t w1 = smem_u32(s_w), w2 = w1 + S::W1_BYTES, w3 = w2 + HM * S::W2_BYTES;
    // descriptors advance by (bytes >> 4) in their low 14-bit start-address field
    const uint64_t d_w1 = umma_desc_k_sw128(w1), d_w2 = umma_desc_k_sw128(w2), d_w3 = umma_desc_k_sw128(w3);
    const uint64_t d_ones = umma_desc_k_sw32(smem_u32(s_ones));
    // the K columns past 64 of W1 (K1 > 64): SW32 / SW64 part after W1's SW128 atom
    const uint64_t d_w1b = S::K2B == 64 ? umma_desc_k_sw64(w1 + 64 * 128) : umma_desc_k_sw32(w1 + 64 * 128);
    // Operand hand-off to the MMA issuer: three warps of the warpgroup only arrive on the
    // context's named barrier (bar.arrive) and move on to the other context; the issuing
    // warp waits (bar.sync) and issues.  One barrier id per context keeps successive phases
    // apart.  The issuing warp rotates with (warpgroup, context) so the MMA-issue work is
    // spread over the four SM sub-partitions instead of piling up on warp 0's.
    auto handoff = [&](const Ctx<P>& C) {
        if (q == C.iq)
            named_bar_sync(1 + wg * NC + C.id, 128);
        else
            named_bar_arrive(1 + wg * NC + C.id, 128);
    };
    constexpr uint32_t ID64 = idesc_f16(128, 64), ID16 = idesc_f16(128, 16);
    // MMA issue: whole warp (elect.sync) when the operands are provably warp-uniform
    // (DECODE_WARP_ALL: also the instantiations whose operands are not provably uniform; ptxas
    // then broadcasts them from the elected lane -- A/B: random queries 20.5 -> 18.5, off)
    constexpr bool WI = DECODE_WARP_ISSUE && (UNI || DECODE_WARP_ALL);
    constexpr bool WG4 = WI && DECODE_WARP_ISSUE >= 2;  // whole layers as one asm block
    auto mma = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
        if constexpr (WI)
            mma_f16_ss_warp(d, a, b, id, acc);
        else
            mma_f16_ss(d, a, b, id, acc);
    };
    auto commit = [&](uint64_t* bar) {
        if constexpr (WI)
            mma_commit_warp(bar);
        else
            mma_commit(bar);
    };
    // single material: tiles blockIdx-strided over [first, ntiles); multi: per-run ranges
    int ntiles = TILED || p.mode == 0 ? p.n_tiles : (int)((p.nq + TILE_M - 1) / TILE_M);
    int stride = (int)gridDim.x * NW * NC;  // tiles advance by NC contexts per warpgroup
    Run R;
    R.grids = nullptr;
    R.b3 = nullptr;
    R.perm = MULTI ? mt->perm : nullptr;
    R.ts0 = R.seg0 = R.cnt = 0;

    Ctx<P> cx[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        cx[c].phase = 0;
        cx[c].abuf = smem_u32(s_a + (wg * NC + c) * S::ABUF);
        cx[c].tcol = tmem + (uint32_t)((wg * NC + c) * 64);
        cx[c].bar = &s_bar[wg * NC + c];
        cx[c].id = c;
        cx[c].iq = (wg * NC + c) & 3;
        cx[c].adesc = umma_desc_k_sw128(cx[c].abuf);
        cx[c].stage = smem_u32(s_stage + (wg * NC + c) * S::STAGE);
        cx[c].ptile = -1;
        if (!MULTI) {
            cx[c].tile = (TILED || p.mode == 0 ? p.tile_first : 0) + ((int)blockIdx.x * NW + wg) * NC + c;
            if (cx[c].tile < ntiles) fetch_tile<P, MULTI, CT, TILED>(p, R, cx[c].tile, row, cx[c].nxt);
        }
    }

    // P0: assemble X of the context's tile from its prefetched latents, MMA1, prefetch next
    auto phase0 = [&](Ctx<P>& C) {
        if (C.tile >= ntiles) return;
        {
            uint32_t xw[P::K1W];
            assemble_words<P>(p, s_pe, C.nxt, xw);
            store_row<P::K1W>(C.abuf, row, xw);
        }
        C.dst = C.nxt.dst;
        C.flags = C.nxt.info >> 20;
        fence_proxy_async_smem();
        tc_fence_before();
        handoff(C);
        if (q == C.iq && (WI || lane == 0)) {
            if (TMA && C.ptile >= 0 && lane == 0) {  // the previous tile's staged output: one bulk store
                bulk_s2g(p.out + (int64_t)C.ptile * TILE_M * (CT ? CT : p.c), C.stage, TILE_M * 2 * (CT ? CT : p.c));
                bulk_commit();
            }
            tc_fence_after();
            if constexpr (WG4 && S::K2 == 0) {  // the whole layer in one asm block
                mma4_commit_warp<false>(C.tcol, C.adesc, d_w1, ID64, 0, 0, C.bar);
            } else if constexpr (WG4) {  // K1 > 64: the SW128 atom's chain, then the SW32 / SW64 part
                mma_chain4_warp<2, 2>(C.tcol, C.adesc, d_w1, ID64, 0);
                const uint64_t a2 = S::K2B == 64 ? umma_desc_k_sw64(C.abuf + 128 * 128) : umma_desc_k_sw32(C.abuf + 128 * 128);
                if constexpr (S::K2 == 32) mma_f16_ss_warp(C.tcol, a2, d_w1b, ID64, 1);
                mma1_commit_warp(C.tcol, a2 + (S::K2 == 32 ? 2 : 0), d_w1b + (S::K2 == 32 ? 2 : 0), ID64, 1, C.bar);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) mma(C.tcol, C.adesc + (uint64_t)(k * 2), d_w1 + (uint64_t)(k * 2), ID64, k > 0);
                if constexpr (S::K2 > 0) {  // K columns 64 .. K1 - 1 from the SW32 / SW64 parts
                    const uint64_t a2 =
                        S::K2B == 64 ? umma_desc_k_sw64(C.abuf + 128 * 128) : umma_desc_k_sw32(C.abuf + 128 * 128);
#pragma unroll
                    for (int k = 0; k < S::K2 / 16; ++k) mma(C.tcol, a2 + (uint64_t)(k * 2), d_w1b + (uint64_t)(k * 2), ID64, 1);
                }
                commit(C.bar);
            }
        }
        C.ptile = -1;
        if (DECODE_FETCH_AT == 0) {
            const int nt = C.tile + stride;
            if (nt < ntiles) fetch_tile<P, MULTI, CT, TILED>(p, R, nt, row, C.nxt);  // loads overlap the MLP
        }
    };
    // P1..P(HM+1): wait for the previous MMA, epilogue to the A tile, next layer's MMA
    // chk = false: the caller knows the context holds a tile (steady-state loop below)
    auto phase_hidden = [&](Ctx<P>& C, int layer, bool chk) {
        if (chk && C.tile >= ntiles) return;
        if (DECODE_FETCH_AT == 1 && layer == 1) {
            const int nt = C.tile + stride;
            if (nt < ntiles) fetch_tile<P, MULTI, CT, TILED>(p, R, nt, row, C.nxt);  // fills the MMA wait
        }
        mbar_wait(C.bar, C.phase);
        C.phase ^= 1;
        tc_fence_after();
        // pipelined TMEM loads for NTC 0.2 mip tiles (+4.9% on the headline chain); the query
        // and multi-material instantiations measured neutral / -2.4% with them, the two-
        // warpgroup K1 > 64 profiles (255 registers, no spills to remove) about -1.5%
        epilogue_hidden<ACT, UNI>(C.tcol + lane_off, C.abuf, row);
        fence_proxy_async_smem();
        tc_fence_before();
        handoff(C);
        if (q == C.iq && (WI || lane == 0)) {
            tc_fence_after();
            const bool last = layer == HM;
            // the staging buffer is rewritten once this context's output MMA completes: its
            // previous bulk store must have read it (issued two phases ago, normally done)
            if (TMA && last && lane == 0) bulk_wait_read0();
            const uint64_t dl = last ? d_w3 : d_w2 + (uint64_t)((layer * S::W2_BYTES) >> 4);
            const uint32_t id = last ? ID16 : ID64;
            // hidden-layer bias: one K=16 MMA of the ones tile against the layer's SW32 bias
            // atom; the output bias is added in the output epilogue (FADD.SAT, free with the clamp)
            if constexpr (WG4) {
                if (last)
                    mma4_commit_warp<false>(C.tcol, C.adesc, dl, id, 0, 0, C.bar);
                else
                    mma4_commit_warp<true>(C.tcol, C.adesc, dl, id, d_ones,
                                           umma_desc_k_sw32(w2 + layer * S::W2_BYTES + 64 * 128), C.bar);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) mma(C.tcol, C.adesc + 2 * k, dl + 2 * k, id, k > 0);
                if (!last) mma(C.tcol, d_ones, umma_desc_k_sw32(w2 + layer * S::W2_BYTES + 64 * 128), id, 1);
                commit(C.bar);
            }
        }
    };
    // P(HM+2): wait for the output MMA, clamp, store, then start the context's next tile
    auto phase_out = [&](Ctx<P>& C, bool chk) {
        if (chk && C.tile >= ntiles) return;
        mbar_wait(C.bar, C.phase);
        C.phase ^= 1;
        tc_fence_after();
        uint32_t r[16];
        tmem_ld16(C.tcol + lane_off, r);
        tmem_wait_ld();
        uint32_t o[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] = 0u;
#pragma unroll
        for (int k = 0; k < (CT ? (CT + 1) / 2 : 8); ++k)
            o[k] = pack_half2(__saturatef(__uint_as_float(r[2 * k]) + (MULTI ? R.b3 : p.b3)[2 * k]),
                              __saturatef(__uint_as_float(r[2 * k + 1]) + (MULTI ? R.b3 : p.b3)[2 * k + 1]));
        if (TMA && C.tile < p.tma_tiles) {  // whole tile: rows into SMEM, stored by the next phase0
            uint16_t* sdst = reinterpret_cast<uint16_t*>(s_stage + (size_t)(wg * NC + C.id) * S::STAGE) +
                             row * (CT ? CT : p.c);
            store_output<CT, TILED>(p, sdst, true, false, (CT ? CT : p.c) & 1, row, o);  // R13: clamp [0,1]
            C.ptile = C.tile;
        } else {
            store_output<CT, TILED>(p, C.dst, C.flags & 1, C.flags & 2, !MULTI && C.tile < p.pair_tiles, row, o);
        }
        tc_fence_before();
        C.tile += stride;
        phase0(C);
    };

    // tiles first + 2 wg + c, advancing by `stride`, up to `ntiles` (exclusive), through the
    // two-context pipeline; returns with every context drained (all MMAs waited for)
    auto run = [&](int first) {
        if (MULTI) {
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                cx[c].tile = first + wg * NC + c;
                if (cx[c].tile < ntiles) fetch_tile<P, MULTI, CT, TILED>(p, R, cx[c].tile, row, cx[c].nxt);
            }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) phase0(cx[c]);
        auto busy = [&]() {
            bool b = false;
#pragma unroll
            for (int c = 0; c < NC; ++c) b = b || cx[c].tile < ntiles;
            return b;
        };
        // steady state: every context holds a tile (the last context's is the largest), so the
        // phases skip their idle checks; the tail rounds check per context
        if (DECODE_STEADY)
            while (cx[NC - 1].tile < ntiles) {
#pragma unroll
                for (int layer = 0; layer <= HM; ++layer) {
#pragma unroll
                    for (int c = 0; c < NC; ++c) phase_hidden(cx[c], layer, false);
                }
#pragma unroll
                for (int c = 0; c < NC; ++c) phase_out(cx[c], false);
            }
        while (busy()) {
#pragma unroll
            for (int layer = 0; layer <= HM; ++layer) {
#pragma unroll
                for (int c = 0; c < NC; ++c) phase_hidden(cx[c], layer, true);
            }
#pragma unroll
            for (int c = 0; c < NC; ++c) phase_out(cx[c], true);
        }
    };
    if constexpr (!MULTI) {
        run(0);  // tiles and their first fetches were set up with the contexts
        if constexpr (TMA) {  // each context's last staged tile (its phase0 found no next tile)
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                if (cx[c].ptile < 0) continue;
                fence_proxy_async_smem();
                handoff(cx[c]);
                if (q == cx[c].iq && lane == 0) {
                    bulk_s2g(p.out + (int64_t)cx[c].ptile * TILE_M * (CT ? CT : p.c), cx[c].stage,
                             TILE_M * 2 * (CT ? CT : p.c));
                    bulk_commit();
                }
            }
            if (lane == 0) bulk_wait0();  // every bulk store complete before the CTA exits
        }
    } else {
        // a contiguous share of the material-sorted tile list; one weight image at a time
        const int T = __ldg(mt->tstart + mt->n_mats);
        const int c0 = (int)((int64_t)T * blockIdx.x / gridDim.x), c1 = (int)((int64_t)T * (blockIdx.x + 1) / gridDim.x);
        int m = 0;
        while (m < mt->n_mats && __ldg(mt->tstart + m + 1) <= c0) ++m;
        for (int pos = c0; pos < c1 && m < mt->n_mats; ++m) {
            const int ts1 = __ldg(mt->tstart + m + 1), e = min(c1, ts1);
            if (e <= pos) continue;
            // the previous run is drained: its MMAs no longer read the weight image
            __syncthreads();
            const uint4* wsrc = mt->rec[m].wimg;
            for (uint32_t i = tid; i < S::WIMG / 16; i += blockDim.x) reinterpret_cast<uint4*>(s_w)[i] = __ldg(wsrc + i);
            fence_proxy_async_smem();
            __syncthreads();
            R.grids = mt->rec[m].grids;
            R.b3 = mt->rec[m].b3;
            R.ts0 = __ldg(mt->tstart + m);
            R.seg0 = __ldg(mt->seg + m);
            R.cnt = __ldg(mt->seg + m + 1) - R.seg0;
            ntiles = e;
            stride = NW * NC;
            run(pos);
            pos = e;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

template <class P, int HM, int ACT, int CT = 0, bool TILED = false>
__global__ void __launch_bounds__(DecodeSmem<P, HM>::NWG * 128, 1) decode_kernel(const __grid_constant__ DecodeParams p) {
    decode_body<P, HM, false, ACT, CT, TILED>(p, nullptr);
}

template <class P, int HM, int ACT, int CT = 0>
__global__ void __launch_bounds__(DecodeSmem<P, HM>::NWG * 128, 1)
    decode_multi_kernel(const __grid_constant__ DecodeParams p, const __grid_constant__ MultiTable mt) {
    decode_body<P, HM, true, ACT, CT>(p, &mt);
}

// Tests only: the same addressing + assembly, written to global memory in canonical order.
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
    Fetch<P> f;
    fetch_texel<P>(p, p.grids, m, x, y, f, p.dbg_addr + i * 17);
    uint32_t w[P::K1W];
    assemble_words<P>(p, s_pe, f, w);
    uint16_t* X = p.dbg_X + i * P::D;
    for (int k = 0; k < P::D; ++k) X[canonical_col<P>(k)] = (uint16_t)(w[k >> 1] >> (16 * (k & 1)));
}

// Weight image (global copy of the SMEM layout): W1's K columns [0, 64) as one SW128 atom of
// 64 rows (G0 columns permuted like X, b1 at column D) and, for K1 > 64, the columns past 64
// as an SW32 / SW64 part; per hidden layer an SW128 weights atom and an SW32 bias atom
// (column 0 = b); W3 (16 rows) and its bias atom.
template <class P, int HM>
__device__ __forceinline__ uint32_t wimg_w1_offset(int r, int k) {
    using S = DecodeSmem<P, HM>;
    if (k < 64) return sw128_offset(r, k);
    return 64 * 128 + (S::K2B == 64 ? sw64_offset(r, k - 64) : sw32_offset(r, k - 64));
}
template <class P, int HM>
constexpr int wimg_items() {
    return 64 * P::K1 + HM * (64 * 64 + 64 * 16) + 2 * 16 * 64;
}
template <class P, int HM>
__global__ void wimg_kernel(const uint16_t* __restrict__ w, int c, uint8_t* __restrict__ img) {
    using S = DecodeSmem<P, HM>;
    constexpr int D = P::D, n1 = 64 * P::K1, n2 = 64 * 64 + 64 * 16, n3 = 2 * 16 * 64;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n1 + HM * n2 + n3) return;
    const int P1 = D * HID, P2 = HID * HID;
    uint16_t v = 0;
    uint32_t off;
    if (i < n1) {
        const int r = i / P::K1, k = i % P::K1;
        if (k < D) v = w[r * D + canonical_col<P>(k)];
        else if (k == D) v = w[P1 + r];
        off = wimg_w1_offset<P, HM>(r, k);
    } else if (i < n1 + HM * n2) {
        const int l = (i - n1) / n2, e = (i - n1) % n2;
        const int base = P1 + HID + l * (P2 + HID);
        if (e < 4096) {
            const int r = e / 64, k = e % 64;
            v = w[base + r * HID + k];
            off = S::W1_BYTES + l * S::W2_BYTES + sw128_offset(r, k);
        } else {
            const int r = (e - 4096) / 16, k = (e - 4096) % 16;
            v = k == 0 ? w[base + P2 + r] : (uint16_t)0;
            off = S::W1_BYTES + l * S::W2_BYTES + 64 * 128 + sw32_offset(r, k);
        }
    } else {
        const int e = i - n1 - HM * n2, bias = e / 1024, r = (e % 1024) / 64, k = e % 64;
        const int base = P1 + HID + HM * (P2 + HID);
        if (r < c) v = bias ? (k == 0 ? w[base + HID * c + r] : (uint16_t)0) : w[base + r * HID + k];
        off = S::W1_BYTES + HM * S::W2_BYTES + bias * 2048 + sw128_offset(r, k);
    }
    *reinterpret_cast<uint16_t*>(img + off) = v;
}

// ------------------------------------------------------------------ launchers
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

template <class F>
static auto dispatch(int pid, int hm, F&& f) {
    switch (pid * 2 + (hm - 1)) {
        case 0: return f(NTC02{}, std::integral_constant<int, 1>{});
        case 1: return f(NTC02{}, std::integral_constant<int, 2>{});
        case 2: return f(NTC05{}, std::integral_constant<int, 1>{});
        case 3: return f(NTC05{}, std::integral_constant<int, 2>{});
        case 4: return f(NTC10{}, std::integral_constant<int, 1>{});
        case 5: return f(NTC10{}, std::integral_constant<int, 2>{});
        case 6: return f(NTC225{}, std::integral_constant<int, 1>{});
        default: return f(NTC225{}, std::integral_constant<int, 2>{});
    }
}

// + the activation (0 hardGELU, 1 exact GELU) for the decode kernels
template <class F>
static auto dispatch_act(int pid, int hm, int act, F&& f) {
    return dispatch(pid, hm, [&](auto pr, auto h) {
        if (act == 1) return f(pr, h, std::integral_constant<int, 1>{});
        return f(pr, h, std::integral_constant<int, 0>{});
    });
}

uint32_t decode_wimg_bytes(int pid, int hm) {
    return dispatch(pid, hm, [](auto pr, auto h) { return DecodeSmem<decltype(pr), decltype(h)::value>::WIMG; });
}

cudaError_t build_wimg(int pid, int hm, const uint16_t* w, int c, uint8_t* img, cudaStream_t s) {
    return dispatch(pid, hm, [&](auto pr, auto h) {
        using PP = decltype(pr);
        constexpr int HMv = decltype(h)::value;
        const int n = wimg_items<PP, HMv>();
        wimg_kernel<PP, HMv><<<(n + 255) / 256, 256, 0, s>>>(w, c, img);
        return cudaGetLastError();
    });
}

cudaError_t launch_decode(int pid, int hm, const DecodeParams& p, int grid, cudaStream_t s) {
    return dispatch_act(pid, hm, p.act, [&](auto pr, auto h, auto a) {
        using PP = decltype(pr);
        constexpr int HMv = decltype(h)::value;
        using SS = DecodeSmem<PP, HMv>;
        // mip tiles (mode 0) run an instantiation compiled for that mode (no query branches,
        // uniform-register MMA issue); queries the general one
        auto* k = p.mode == 0 ? decode_kernel<PP, HMv, decltype(a)::value, 0, true>
                              : decode_kernel<PP, HMv, decltype(a)::value>;
        // the bench's headline material (NTC 0.2, [57,64,64,9], hardGELU) gets its channel
        // count (and, for mip tiles, the mode) compiled into the kernel
        if constexpr (std::is_same<PP, NTC02>::value && HMv == 1 && decltype(a)::value == 0)
            if (p.c == 9) k = p.mode == 0 ? decode_kernel<PP, HMv, 0, 9, true> : decode_kernel<PP, HMv, 0, 9>;
        // and the 16-channel material of the random-access line (configs[2])
        if constexpr (std::is_same<PP, NTC02>::value && HMv == 1 && decltype(a)::value == 0)
            if (p.c == 16) k = p.mode == 0 ? decode_kernel<PP, HMv, 0, 16, true> : decode_kernel<PP, HMv, 0, 16>;
        cudaError_t e = ensure_smem((const void*)k, SS::BYTES);
        if (e != cudaSuccess) return e;
        k<<<grid, SS::NWG * 128, SS::BYTES, s>>>(p);
        return cudaGetLastError();
    });
}

cudaError_t launch_decode_multi(int pid, int hm, const DecodeParams& p, const MultiTable& mt, int grid,
                                cudaStream_t s) {
    return dispatch_act(pid, hm, p.act, [&](auto pr, auto h, auto a) {
        using PP = decltype(pr);
        constexpr int HMv = decltype(h)::value;
        using SS = DecodeSmem<PP, HMv>;
        auto* k = decode_multi_kernel<PP, HMv, decltype(a)::value>;
        // the 8-channel materials of the multi-material line (Table 4 analog)
        if constexpr (std::is_same<PP, NTC02>::value && HMv == 1 && decltype(a)::value == 0)
            if (p.c == 8) k = decode_multi_kernel<PP, HMv, 0, 8>;
        cudaError_t e = ensure_smem((const void*)k, SS::BYTES);
        if (e != cudaSuccess) return e;
        k<<<grid, SS::NWG * 128, SS::BYTES, s>>>(p, mt);
        return cudaGetLastError();
    });
}

cudaError_t launch_debug_assemble(int pid, const DecodeParams& p, cudaStream_t s) {
    return dispatch(pid, 1, [&](auto pr, auto) {
        using PP = decltype(pr);
        const int64_t blocks = (p.nq + 127) / 128;
        debug_assemble_kernel<PP><<<(unsigned)blocks, 128, 0, s>>>(p);
        return cudaGetLastError();
    });
}

}  // namespace ntc
