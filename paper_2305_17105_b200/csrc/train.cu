// train.cu -- NTC compression training step on sm_100a (tcgen05 + TMEM), product code.
//
// ntc_train_step(GRADS):
//   prep_kernel      t2: noisy latents (Philox U(-Q/2,Q/2)) and zeroed latent
//                    gradients over the batch footprint (disjoint boxes)
//   train_kernel     t1,t3-t7: per 128-texel tile: fp16 input assembly from the noisy fp32
//                    latents, forward MLP on tcgen05 (Z kept as fp16 hardGELU' tiles), mean-L2
//                    loss, backward MMAs (dH2 = d3 W3, dH1 = d2 W2, dX = d1 W1), weight
//                    gradients accumulated in TMEM across the CTA's tiles as two stacked
//                    MN-major MMAs, latent-gradient scatter with vector reductions
//   reduce_kernel    t6: fixed-order sum of the per-warpgroup weight-gradient partials, loss
// ntc_train_step(APPLY):
//   adam_kernel      t8: Adam on the weights (dense) and on the footprint latents (sparse:
//                    g == 0 skipped, R18), then the latent clamp
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "ptx.cuh"

namespace ntc {

constexpr int MAX_BOXES = 256;

// phase of slot 0's first tile after which slot 1 starts (3: after the H1 epilogue, 5: after
// the H2 epilogue, 7: after the loss; 0: both slots start together) -- see train_kernel
#ifndef TRAIN_DESYNC
#define TRAIN_DESYNC 5
#endif
// 1: the backward MMAs (dH = delta W, dX = delta1 W1) accumulate in fp16 -- the delta epilogue
// multiplies fp16(dH) by hardGELU' anyway, so it reads packed half2 words (no conversions), and
// the latent-gradient run sums of the scatter run on half2 words (half the shuffles and adds);
// 0: fp32 accumulators converted in the epilogues
// 1: the output layer's weight-gradient MMAs (dW3/db3, 8 small MMAs) are issued with dH_last
// instead of with dX, so fewer MMAs queue behind dX at the end of the tile
#ifndef TRAIN_DWB_EARLY
#define TRAIN_DWB_EARLY 0
#endif
// 1: prep_kernel is launched with programmatic dependent launch too (griddepcontrol.wait
// before it reads the latents and weights the previous step's Adam wrote)
#ifndef TRAIN_PREP_PDL
#define TRAIN_PREP_PDL 1
#endif
// 1: the training input's G1 bilinear in packed fp16 (HFMA2) instead of fp32 + one rounding
// (A/B: 63.2 vs 62.9 us per C4 step, off)
#ifndef TRAIN_G1_H2
#define TRAIN_G1_H2 0
#endif
// 1 (see train_kernel): A/B, 3 rounds: C4 step 62.9 -> 60.9 us; ptxas: R2UR 56 -> 4, VOTEU 75 -> 6
#ifndef TRAIN_UNI_WARP
#define TRAIN_UNI_WARP 1
#endif
#ifndef TRAIN_WARP_ISSUE  // see train_kernel
#define TRAIN_WARP_ISSUE 2
#endif
#ifndef TRAIN_BWD_F16
#define TRAIN_BWD_F16 1
#endif

struct Box {        // inclusive cell ranges of one grid
    int64_t off;    // element offset of the grid in the canonical latent array
    int32_t r, C, bits;
    int32_t x0, y0, x1, y1;
};

struct TrainParams {
    // geometry of the batch mip
    int32_t W, c, M, mip, lw;
    int32_t r0, r1, lr0, lr1;
    int64_t off0, off1;
    uint32_t lod_word;
    uint32_t pe_words[8][4];
    // batch
    int32_t n_crops;
    int32_t crop[NTC_MAX_CROPS][4];
    int32_t tile_start[NTC_MAX_CROPS + 1];
    int32_t n_tiles;
    const uint16_t* ref;
    int64_t ref_stride;
    float inv_bc;
    // buffers
    const __half* noisy;
    float* grad_lat;
    const uint8_t* wimg;  // fp16 weight image (TrainSmem layout, WEND bytes)
    float* partial;     // [grid][Pst]
    float* loss_partial;  // [grid * slots]
    int32_t P;
    int32_t Pst;          // partial stride: P rounded up to 4 floats (16-byte stores)
    int32_t freeze;       // frozen phase: no latent gradients
};

// ------------------------------------------------------------------ Philox noise (R16)
__device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t b) { return __umulhi(a, b); }

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = mulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = mulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

struct PrepParams {
    Box box[MAX_BOXES];
    int32_t nbox;
    int32_t box_start[MAX_BOXES + 1];  // prefix of latents per box
    const float* latents;
    __half* noisy;  // fp16 noisy latents (the fp16 network-input format, R14)
    float* grad_lat;
    uint64_t seed;
    uint32_t step;
    int32_t noise_on;
    // fp16 weight image of the master weights, built by the trailing blocks of the same launch
    int32_t prep_blocks;  // blocks [0, prep_blocks) do t2; the rest build the image
    const float* params;
    int32_t D, c, hm;
    uint8_t* wimg;
};

// Latents per thread of the footprint-box kernels (prep, latent Adam): consecutive flat
// indices are mostly consecutive latents of one box row, so one box lookup (and, for the
// noise, one Philox block per 4 latents, R16) serves several latents.
constexpr int LPT = 4;

// flat index -> box, latent index, position in the box row and the row length
__device__ __forceinline__ void box_locate_row(const Box* box, const int32_t* start, int nbox, int32_t i, int& b,
                                               int64_t& li, int32_t& rem, int32_t& w) {
    b = 0;
    while (b + 1 < nbox && i >= start[b + 1]) ++b;
    const Box& B = box[b];
    const int32_t k = i - start[b];
    w = (B.x1 - B.x0 + 1) * B.C;
    const int32_t yy = B.y0 + k / w;
    rem = k % w;
    li = B.off + ((int64_t)yy * B.r + B.x0) * B.C + rem;
}

// advance a box cursor from flat index i - 1 to i
__device__ __forceinline__ void box_next(const Box* box, const int32_t* start, int nbox, int32_t i, int& b,
                                         int64_t& li, int32_t& rem, int32_t& w) {
    if (rem + 1 < w && i < start[b + 1]) {
        ++li;
        ++rem;
    } else {
        box_locate_row(box, start, nbox, i, b, li, rem, w);
    }
}

__device__ __forceinline__ void box_locate(const Box* box, const int32_t* start, int nbox, int32_t i, int& b,
                                           int64_t& li) {
    b = 0;
    while (b + 1 < nbox && i >= start[b + 1]) ++b;
    const Box& B = box[b];
    const int32_t k = i - start[b];
    const int32_t w = (B.x1 - B.x0 + 1) * B.C;
    const int32_t yy = B.y0 + k / w, rem = k % w;
    li = B.off + ((int64_t)yy * B.r + B.x0) * B.C + rem;
}

#ifdef NTC_TRAIN_TRACE
// phase timestamps of the MMA-issuing thread of every slot (tools/trace_train.py only; the
// product library is built without NTC_TRAIN_TRACE): [cta][slot][iteration < 16][warp][32] clocks;
// k < 16 after a phase boundary, 16 + k when the warp arrives at the barrier that ends phase k
__device__ uint32_t* g_trace;
extern "C" void ntc_trace_set(uint32_t* p) { cudaMemcpyToSymbol(g_trace, &p, sizeof p); }
#define NTC_TRACE(k)                                                                                          \
    do {                                                                                                     \
        if (lane == 0 && g_trace && iter < 16)                                                               \
            g_trace[((((size_t)blockIdx.x * SLOTS + slot) * 16 + iter) * 8 + (warp & 7)) * 32 + (k)] =         \
                (uint32_t)clock64();                                                                         \
    } while (0)
__device__ __forceinline__ uint32_t gtimer_lo() {
    uint32_t t;
    asm volatile("mov.u32 %0, %%globaltimer_lo;" : "=r"(t));
    return t;
}
// kernel-level stamps in iteration slot 15: 0 entry, 1 after the prologue, 2 after the tile
// loop, 3 exit (clock64); 4 entry, 5 exit (%globaltimer, ns)
#define NTC_TRACE_K(k, v)                                                                                     \
    do {                                                                                                     \
        if (lane == 0 && g_trace)                                                                            \
            g_trace[((((size_t)blockIdx.x * SLOTS + (warp >> 3)) * 16 + 15) * 8 + (warp & 7)) * 32 + (k)] = (v); \
    } while (0)
#else
#define NTC_TRACE_K(k, v) \
    do {                  \
    } while (0)
#define NTC_TRACE(k) \
    do {             \
    } while (0)
#endif

// ------------------------------------------------------------------ fused forward + backward
// SMEM layout for depth HM (1: [D,64,64,c]; 2: [D,64,64,64,c], R11) and KA 64-column K atoms
// of X (1: K1 = 64, NTC 0.2; 2: K1 = 80/96, the other Table 2 profiles): fp16 weight images
// (W1 in KA atoms with b1 at column D, W2, [W2b], W3 with 16 rows), a constant ones tile and the
// bias atoms of b2, [b2b], b3 (SW32 K = 16 tiles: the biases enter the accumulators as one extra
// K = 16 MMA of ones x bias, so no epilogue adds them); then per tile pipeline ("slot") the
// SW128 activation tiles.  Only the depth-1 K1 = 64 layout leaves SMEM for two slots.
template <int HM, int KA = 1>
struct TrainSmemT {
    static constexpr uint32_t W1 = 0, W2 = 8192u * KA, W2B = W2 + 8192, W3 = W2 + 8192u * HM;
    static constexpr uint32_t ONES = W3 + 2048;   // [128][16] fp16 SW32, column 0 = 1
    static constexpr uint32_t B2A = ONES + 4096;  // [64][16] SW32, column 0 = b2 (then b2b)
    static constexpr uint32_t B3A = B2A + 2048u * HM;  // [16][16] SW32, column 0 = b3
    static constexpr uint32_t WEND = ((B3A + 512 + 1023) / 1024) * 1024;
    static constexpr uint32_t TILE = 128 * 128;  // one 128 x 64 fp16 SW128 tile
    // depth 1: X[KA] H1 H2 G1 G2 D3; depth 2: X[KA] H1 H2 H3 G1 G2 G3 D3
    // (G1 and G2 adjacent: [delta1 | delta2] is one N=128 operand of the weight-gradient MMA)
    enum {
        X = 0, H1 = KA, H2 = KA + 1, H3 = KA + 2, G1 = KA + 1 + HM, G2 = KA + 2 + HM, G3 = KA + 5,
        D3 = KA + 2 + 2 * HM, NT = KA + 3 + 2 * HM
    };
    static constexpr int SLOTS = (HM == 1 && KA == 1) ? 2 : 1;
    static constexpr uint32_t WG_BYTES = NT * TILE;
    static constexpr uint32_t MISC = 256 + 16 * NTC_MAX_CROPS + 4 * (NTC_MAX_CROPS + 1) + 4 * NTC_MAX_CROPS + 12;
    static constexpr uint32_t BYTES = 1024 + WEND + SLOTS * WG_BYTES + MISC;
    static_assert(BYTES <= 232448, "training SMEM layout exceeds 227 KB");
};
using TrainSmem = TrainSmemT<1>;
constexpr uint32_t TRAIN_WEND_MAX = TrainSmemT<2, 2>::WEND;

__device__ __forceinline__ void sts_row_chunk(uint32_t tile, int row, int chunk, uint32_t a, uint32_t b, uint32_t c,
                                              uint32_t d) {
    sts128(tile + (uint32_t)row * 128u + ((uint32_t)(chunk ^ (row & 7)) << 4), a, b, c, d);
}

__device__ __forceinline__ uint4 lds_row_chunk(uint32_t tile, int row, int chunk) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(tile + (uint32_t)row * 128u + ((uint32_t)(chunk ^ (row & 7)) << 4)));
    return v;
}

__device__ __forceinline__ float hgelu(float z) { return z * __saturatef(fmaf(z, 1.0f / 3.0f, 0.5f)); }
// R15: derivative of the piecewise hardGELU, the middle piece at +-3/2 (decided in fp32: the
// derivative jumps at +-3/2, so the branch must follow the fp32 pre-activation exactly)
__device__ __forceinline__ float hgelu_d(float z) {
    const float t = fmaf(z, 2.0f / 3.0f, 0.5f);
    return z > 1.5f ? 1.0f : (z < -1.5f ? 0.0f : t);
}

__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}

__device__ __forceinline__ void red_add_v2(float* p, float a, float b) {
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}

__device__ __forceinline__ uint32_t h2u(float a, float b) { return pack_half2(a, b); }

// fp16 weight image of the current fp32 master weights (t3), the SMEM layout copied verbatim:
// W1 (+ b1 at column D, it multiplies X's constant 1), W2, [W2b], W3 (16 rows) as SW128
// K-major atoms; the ones tile and the bias atoms b2, [b2b], b3 (column 0, SW32) -- the biases
// take their fp16 rounding like every weight (R14).  ABI parameter order: W1, b1, W2, b2,
// [W2b, b2b], W3, b3.  One item = one fp16 element.
__host__ __device__ constexpr int wimg_items(int hm, int ka) {
    return (ka + hm) * 4096 + 1024 + 2048 + 1024 * hm + 256;
}
template <int HM, int KA>
__device__ __forceinline__ void train_wimg_item_t(int i, const float* __restrict__ w, int D, int c,
                                                  uint8_t* __restrict__ img) {
    using S = TrainSmemT<HM, KA>;
    if (i >= wimg_items(HM, KA)) return;
    const int P1 = D * HID;                            // b1
    const int o3 = P1 + HID + HM * (HID * HID + HID);  // W3
    float v = 0.0f;
    uint32_t off;
    if (i < (KA + HM) * 4096) {
        const int part = i / 4096, e = i % 4096, r = e / 64, kk = e % 64;
        if (part < KA) {  // W1 atom `part`: X features 64 part + kk
            const int k = 64 * part + kk;
            v = k < D ? w[r * D + k] : (k == D ? w[P1 + r] : 0.0f);
            off = S::W1 + 8192u * part + sw128_offset(r, kk);
        } else {          // hidden matrix l
            const int l = part - KA;
            v = w[P1 + HID + l * (HID * HID + HID) + r * HID + kk];
            off = (l == 0 ? S::W2 : S::W2B) + sw128_offset(r, kk);
        }
    } else if ((i -= (KA + HM) * 4096) < 1024) {  // W3, 16 rows (c used)
        const int r = i / 64, kk = i % 64;
        v = r < c ? w[o3 + r * HID + kk] : 0.0f;
        off = S::W3 + sw128_offset(r, kk);
    } else if ((i -= 1024) < 2048) {  // ones tile: column 0 = 1
        const int r = i / 16, kk = i % 16;
        v = kk == 0 ? 1.0f : 0.0f;
        off = S::ONES + sw32_offset(r, kk);
    } else if ((i -= 2048) < 1024 * HM) {  // hidden bias atoms: row j column 0 = b2[j] (b2b)
        const int l = i / 1024, r = (i % 1024) / 16, kk = i % 16;
        v = kk == 0 ? w[P1 + HID + l * (HID * HID + HID) + HID * HID + r] : 0.0f;
        off = S::B2A + 2048u * l + sw32_offset(r, kk);
    } else {  // b3 atom (16 rows, c used)
        i -= 1024 * HM;
        const int r = i / 16, kk = i % 16;
        v = (kk == 0 && r < c) ? w[o3 + HID * c + r] : 0.0f;
        off = S::B3A + sw32_offset(r, kk);
    }
    *reinterpret_cast<__half*>(img + off) = __float2half_rn(v);
}

// t2: noisy = latent + U(-Q/2, Q/2) (one draw per latent per step), grad = 0, over the footprint
__global__ void prep_kernel(const __grid_constant__ PrepParams p) {
    pdl_launch_dependents();  // the training kernel's CTAs may start their prologue meanwhile
    // launched programmatically after the previous step's Adam (TRAIN_PREP_PDL): its latents and
    // weights are complete and visible past this point (a no-op for a plain launch)
    pdl_wait();
    if ((int)blockIdx.x >= p.prep_blocks) {
        const int i = ((int)blockIdx.x - p.prep_blocks) * blockDim.x + threadIdx.x;
        if (p.wimg) {
            const bool ka2 = p.D + 1 > 64;
            if (p.hm == 2)
                ka2 ? train_wimg_item_t<2, 2>(i, p.params, p.D, p.c, p.wimg)
                    : train_wimg_item_t<2, 1>(i, p.params, p.D, p.c, p.wimg);
            else
                ka2 ? train_wimg_item_t<1, 2>(i, p.params, p.D, p.c, p.wimg)
                    : train_wimg_item_t<1, 1>(i, p.params, p.D, p.c, p.wimg);
        }
        return;
    }
    const int32_t n = p.box_start[p.nbox];
    int32_t i = LPT * (int32_t)(blockIdx.x * blockDim.x + threadIdx.x);
    if (i >= n) return;
    int b;
    int64_t li;
    int32_t rem, rw;
    box_locate_row(p.box, p.box_start, p.nbox, i, b, li, rem, rw);
    // all addresses and loads first (the stores below may alias the latents as far as the
    // compiler knows), then the noise and the stores
    int64_t lis[LPT];
    int bs[LPT];
    float vs[LPT];
    const int ne = min(LPT, n - i);
#pragma unroll
    for (int e = 0; e < LPT; ++e) {
        if (e > 0 && e < ne) box_next(p.box, p.box_start, p.nbox, i + e, b, li, rem, rw);
        lis[e] = li;
        bs[e] = b;
        vs[e] = e < ne ? __ldg(p.latents + li) : 0.0f;
    }
    int64_t ctr = -1;
    uint4 r = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int e = 0; e < LPT; ++e) {
        if (e >= ne) break;
        li = lis[e];
        b = bs[e];
        float v = vs[e];
        if (p.noise_on) {
            if ((li >> 2) != ctr) {  // Philox block of latents 4k .. 4k+3 (R16)
                ctr = li >> 2;
                r = philox4x32_10(make_uint4((uint32_t)((uint64_t)li >> 2), (uint32_t)((uint64_t)li >> 34), p.step,
                                             0x4E4F4953u),
                                  make_uint2((uint32_t)p.seed, (uint32_t)(p.seed >> 32)));
            }
            const uint32_t w = (li & 3) == 0 ? r.x : (li & 3) == 1 ? r.y : (li & 3) == 2 ? r.z : r.w;
            // u = (2 (w >> 9) + 1) 2^-24 in (0, 1); noise = (u - 1/2) Q, exact in fp32
            const float u = (float)(2u * (w >> 9) + 1u) * 5.9604644775390625e-8f;
            v += (u - 0.5f) * (1.0f / (float)(1 << p.box[b].bits));
        }
        p.noisy[li] = __float2half_rn(v);
        p.grad_lat[li] = 0.0f;
    }
}

// hidden activation and its derivative: hardGELU (R15) or exact GELU (f4):
// x Phi(x) and Phi(x) + x phi(x)
template <int ACT>
__device__ __forceinline__ void act_and_grad(float z, float& h, float& g) {
    if constexpr (ACT == 0) {
        h = hgelu(z);
        g = hgelu_d(z);
    } else {
        const float Phi = 0.5f * (1.0f + erff(z * 0.70710678118654752f));
        const float phi = 0.39894228040143268f * expf(-0.5f * z * z);
        h = z * Phi;
        g = fmaf(z, phi, Phi);
    }
}

// hardGELU and its derivative (R15) of a column pair, as packed fp16 words.  Outside the
// middle piece s = sat(z/3 + 1/2) is exactly the derivative (0 below -3/2, 1 above +3/2), so
// g = |z| <= 3/2 ? 2z/3 + 1/2 : s (equal to hgelu_d for every finite z); h and t run packed.
__device__ __forceinline__ void hgelu_and_grad2(float z0, float z1, uint32_t& hw, uint32_t& gw) {
    const float2 z = make_float2(z0, z1);
    const float2 s = make_float2(__saturatef(fmaf(z0, 1.0f / 3.0f, 0.5f)), __saturatef(fmaf(z1, 1.0f / 3.0f, 0.5f)));
    const float2 hh = __fmul2_rn(z, s);
    const float2 t = __ffma2_rn(z, make_float2(2.0f / 3.0f, 2.0f / 3.0f), make_float2(0.5f, 0.5f));
    hw = pack_half2(hh.x, hh.y);
    gw = pack_half2(fabsf(z0) <= 1.5f ? t.x : s.x, fabsf(z1) <= 1.5f ? t.y : s.y);
}

template <class P> struct TrainGeom {
    static constexpr int C0 = P::C0, C1 = P::C1;
    static constexpr int D = 4 * C0 + C1 + 13, NLAT = 4 * C0 + C1;
    static constexpr int K1 = ((D + 1 + 15) / 16) * 16, KA = (K1 + 63) / 64;
};

// CT: the channel count as a compile-time constant (0: the runtime p.c) for the reference
// fetch and the loss epilogue
template <class P, int ACT, int HM, int CT = 0>
__global__ void __launch_bounds__(TrainSmemT<HM, TrainGeom<P>::KA>::SLOTS * 256, 1)
    train_kernel(const __grid_constant__ TrainParams p) {
    // Two independent tile pipelines ("slots") per CTA, 8 warps each.  The 4 TMEM lane
    // quarters of a 128-texel tile are served by two warps each that split the columns: half
    // h = 0 owns columns [0, 32) of every 64-wide activation (and the G0 part of X / dX, the
    // reference texels and the loss), half h = 1 columns [32, 64) (and the G1 / PE / LOD part).
    // Depth HM = 2 ([D,64,64,64,c], R11) adds a hidden layer (H3/G3 tiles, one more forward
    // and backward round trip, a third weight-gradient stack) and runs one slot per CTA.
    // KA = 2 (the K1 = 80/96 profiles): X spans two K atoms; the weight gradients of W1 come
    // from the stack [X0^T; X1^T], the biases b2/b2b/b3 through the constant column D in X1.
    using G = TrainGeom<P>;
    constexpr int C0 = G::C0, C1 = G::C1, D = G::D, NLAT = G::NLAT, K1 = G::K1, KA = G::KA;
    using S = TrainSmemT<HM, KA>;
    constexpr int SLOTS = S::SLOTS;
    constexpr int NLATP = ((NLAT + 15) / 16) * 16;  // dX columns (MMA N)
    constexpr int DX = D - 64 * (KA - 1);           // row of the constant column in the stacked X block
    static_assert(C0 % 4 == 0 && C1 % 2 == 0 && NLATP <= 128 && KA <= 2, "training kernel profile");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + S::WEND + SLOTS * S::WG_BYTES);
    float* s_loss = reinterpret_cast<float*>(s_bar + 2 * SLOTS + 2);  // after the weight-copy barrier
    uint32_t* s_pe = reinterpret_cast<uint32_t*>(s_loss + 4);
    uint32_t* s_tmem = s_pe + 32;
    int4* s_crop = reinterpret_cast<int4*>(s_tmem + 4);
    int* s_ts = reinterpret_cast<int*>(s_crop + NTC_MAX_CROPS);
    int* s_csh = s_ts + NTC_MAX_CROPS + 1;  // log2 of the crop width when it is a power of 2, else -1

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    NTC_TRACE_K(0, (uint32_t)clock64());
#ifdef NTC_TRAIN_TRACE
    NTC_TRACE_K(4, gtimer_lo());
#endif
    // slot and the TMEM base go through a shuffle: provably warp-uniform, so the MMA-issuing
    // thread keeps its descriptors in uniform registers (no R2UR waterfall per tcgen05.mma)
    // (with TRAIN_UNI_WARP the column half and lane quarter too: every warp-role test -- the
    // issuing warp, the half -- is then provably warp-uniform, which lets ptxas keep the MMA
    // operands and the role-dependent addresses on the uniform datapath)
    const int slot = __shfl_sync(0xffffffffu, warp >> 3, 0);
    const int wrole = TRAIN_UNI_WARP ? __shfl_sync(0xffffffffu, warp & 7, 0) : warp & 7;
    const int h = wrole >> 2, q = wrole & 3, row = q * 32 + lane;
    const int c = CT ? CT : p.c;

    // ---- weight images (fp16, built once per step by the trailing blocks of prep_kernel; the
    // same images serve the backward MMAs through MN-major descriptors): one bulk TMA copy
    // after the prologue, waited by the MMA-issuing threads only, after the first tile's loads
    uint64_t* s_wbar = s_bar + 2 * SLOTS;
    if (tid < 32) s_pe[tid] = (&p.pe_words[0][0])[tid];
    if (tid < 4) s_loss[tid] = 0.0f;
    if (tid < NTC_MAX_CROPS) {
        s_crop[tid] = make_int4(p.crop[tid][0], p.crop[tid][1], p.crop[tid][2], p.crop[tid][3]);
        const int cw = p.crop[tid][2];
        s_csh[tid] = cw > 0 && (cw & (cw - 1)) == 0 ? __ffs(cw) - 1 : -1;
    }
    if (tid <= NTC_MAX_CROPS) s_ts[tid] = p.tile_start[tid];
    if (tid == 0) {
        for (int i = 0; i < 2 * SLOTS; ++i) mbar_init(&s_bar[i], 1);
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
    // launched programmatically after prep_kernel: the prologue above overlaps prep's tail;
    // its outputs (weight image, noisy latents, zeroed latent gradients) are read only after
    // this wait
    pdl_wait();
    if (tid == 0) {
        mbar_init(s_wbar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(s_wbar, S::WEND);
        bulk_g2s(smem_u32(smem), p.wimg, S::WEND, s_wbar);
    }
    NTC_TRACE_K(1, (uint32_t)clock64());

    // TMEM per slot: depth 1: [0,128) dW-a accumulator, [128,144) dW-b, [192,256) scratch;
    // depth 2: [0,128) dW-a, [128,192) dW-m (the middle layer), [192,208) dW-b, [256,320) scratch
    const uint32_t tbase = __shfl_sync(0xffffffffu, *s_tmem, 0) + (uint32_t)slot * (512u / SLOTS);
    const uint32_t t_acc_a = tbase, t_acc_m = tbase + 128, t_acc_b = tbase + (HM == 1 ? 128 : 192);
    const uint32_t t_s = tbase + (SLOTS == 2 ? 192 : 256);  // 64 (two slots) or 128 scratch columns
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t tiles = sbase + S::WEND + (uint32_t)slot * S::WG_BYTES;
    const uint32_t tX = tiles + S::X * S::TILE, tH1 = tiles + S::H1 * S::TILE, tH2 = tiles + S::H2 * S::TILE;
    const uint32_t tG1 = tiles + S::G1 * S::TILE, tG2 = tiles + S::G2 * S::TILE, tD3 = tiles + S::D3 * S::TILE;
    const uint32_t tH3 = tiles + S::H3 * S::TILE, tG3 = tiles + S::G3 * S::TILE;  // depth 2 only
    const uint32_t tHL = HM == 1 ? tH2 : tH3, tGL = HM == 1 ? tG2 : tG3;        // last hidden layer
    const uint32_t tXB = tX + (uint32_t)(KA - 1) * S::TILE;  // X atom holding the constant column D
    // the two issuing warps sit on different sub-partitions.  TRAIN_WARP_ISSUE 0: lane 0 issues
    // each MMA (a single-thread waterfall around every tcgen05.mma); 1: the whole warp through
    // elect.sync, per MMA (measured slower: 65.5 vs 64.3 us); 2 (default): the whole warp, each
    // MMA group one asm block (one elect per group): 63.2 vs 64.4 us per C4 step (A/B, 3 rounds)
    // TRAIN_WARP_ISSUE = 2: each MMA group as one asm block (every profile and depth)
    constexpr bool CH = TRAIN_WARP_ISSUE >= 2;
    constexpr bool WARP = TRAIN_WARP_ISSUE == 1 || CH;
    const bool issuer = wrole == slot * 2 && (WARP || lane == 0);
    auto mma = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
        if constexpr (WARP)
            mma_f16_ss_warp(d, a, b, id, acc);
        else
            mma_f16_ss(d, a, b, id, acc);
    };
    auto commit = [&](uint64_t* mb) {
        if constexpr (WARP)
            mma_commit_warp(mb);
        else
            mma_commit(mb);
    };
    uint64_t* bar = &s_bar[slot];
    uint64_t* bar2 = &s_bar[SLOTS + slot];
    uint32_t phase = 0, phase2 = 0;
    bool pending_w = false;  // weight-gradient MMAs of the previous tile in flight
    auto sync_slot = [&]() {
        fence_proxy_async_smem();
        tc_fence_before();
        named_bar_sync(1 + slot, 256);
    };
    auto wait_mma = [&]() {
        mbar_wait(bar, phase);
        phase ^= 1;
        tc_fence_after();
    };
    const uint64_t dW1 = umma_desc_k_sw128(sbase + S::W1), dW2 = umma_desc_k_sw128(sbase + S::W2);
    const uint64_t dW3 = umma_desc_k_sw128(sbase + S::W3), dW2B = umma_desc_k_sw128(sbase + S::W2B);
    // bias MMAs: ones[128 x 16] x bias atom^T adds b2 / b2b / b3 to every row of the accumulator
    const uint64_t dONES = umma_desc_k_sw32(sbase + S::ONES), dB2 = umma_desc_k_sw32(sbase + S::B2A);
    const uint64_t dB2B = umma_desc_k_sw32(sbase + S::B2A + 2048), dB3 = umma_desc_k_sw32(sbase + S::B3A);
    const uint64_t dX = umma_desc_k_sw128(tX), dH1 = umma_desc_k_sw128(tH1), dH2 = umma_desc_k_sw128(tH2);
    const uint64_t dG1 = umma_desc_k_sw128(tG1), dG2 = umma_desc_k_sw128(tG2), dD3 = umma_desc_k_sw128(tD3);
    const uint64_t dHL = umma_desc_k_sw128(tHL), dG3 = umma_desc_k_sw128(tG3);
    // MN-major views: W^T operands and the stacked [X^T; H1^T], [X^T; H2^T], delta^T tiles
    const uint64_t mW1 = umma_desc_mn_sw128(sbase + S::W1, 8192), mW2 = umma_desc_mn_sw128(sbase + S::W2, 8192);
    const uint64_t mW3 = umma_desc_mn_sw128(sbase + S::W3, 8192), mW2B = umma_desc_mn_sw128(sbase + S::W2B, 8192);
    const uint64_t mXH1 = umma_desc_mn_sw128(tXB, tH1 - tXB), mXH2 = umma_desc_mn_sw128(tXB, tH2 - tXB);
    const uint64_t mXHL = umma_desc_mn_sw128(tXB, tHL - tXB);
    const uint64_t mXX = umma_desc_mn_sw128(tX, S::TILE);  // KA = 2: [X0^T; X1^T]
    const uint64_t mG1 = umma_desc_mn_sw128(tG1, S::TILE), mG2 = umma_desc_mn_sw128(tG2, S::TILE);
    const uint64_t mG3 = umma_desc_mn_sw128(tG3, S::TILE);
    const uint64_t mD3 = umma_desc_mn_sw128(tD3, S::TILE);
    constexpr uint32_t ID64 = idesc_f16(128, 64), ID16 = idesc_f16(128, 16);
    constexpr bool BF16ACC = TRAIN_BWD_F16 != 0;  // fp16 accumulators of the backward MMAs
    constexpr uint32_t ID64_BT = idesc_f16(128, 64, false, true, !BF16ACC);
    constexpr uint32_t IDX_BT = idesc_f16(128, NLATP, false, true, !BF16ACC);
    constexpr uint32_t ID64_AB = idesc_f16(128, 64, true, true), ID16_AB = idesc_f16(128, 16, true, true);
    constexpr uint32_t ID128_AB = idesc_f16(128, 128, true, true);

    float loss_acc = 0.0f;
    bool first = true;
    const int lw = p.lw;

    // ---- t1/a1: texel of `row` in `tile`, its taps (same integer addressing as decode, R1-R3)
    struct Texel {
        int x, y;
        bool valid;
    };
    auto texel_of = [&](int tile) {
        int k = 0;
        while (tile >= s_ts[k + 1]) ++k;
        const int4 cr = s_crop[k];
        const int li = (tile - s_ts[k]) * TILE_M + row;
        Texel t;
        t.valid = li < cr.z * cr.w;
        const int sh = s_csh[k];  // uniform per tile: power-of-2 crops (the paper's 256^2) shift
        int qx, qy;
        if (sh >= 0) {
            qx = li & (cr.z - 1);
            qy = li >> sh;
        } else {
            qy = li / cr.z;
            qx = li - qy * cr.z;
        }
        t.x = cr.x + (t.valid ? qx : 0);
        t.y = cr.y + (t.valid ? qy : 0);
        return t;
    };
    // G0 taps (half 0) / G1 taps and bilinear weights in 1/256 units (half 1)
    auto taps_g0 = [&](const Texel& t, int (&tx)[2], int (&ty)[2]) {
        const int nx = ((2 * t.x + 1) << p.lr0) - (1 << lw), ny = ((2 * t.y + 1) << p.lr0) - (1 << lw);
        const int i = nx >> (lw + 1), j = ny >> (lw + 1);
        tx[0] = max(i, 0);
        tx[1] = min(i + 1, p.r0 - 1);
        ty[0] = max(j, 0);
        ty[1] = min(j + 1, p.r0 - 1);
    };
    auto taps_g1 = [&](const Texel& t, int (&tx)[2], int (&ty)[2], uint32_t& ax, uint32_t& ay) {
        const int nx = ((2 * t.x + 1) << p.lr1) - (1 << lw), ny = ((2 * t.y + 1) << p.lr1) - (1 << lw);
        const int i = nx >> (lw + 1), j = ny >> (lw + 1);
        const int mask = (2 << lw) - 1;  // exact, see decode
        ax = (uint32_t)(((nx & mask) << 4) >> (lw + 1));
        ay = (uint32_t)(((ny & mask) << 4) >> (lw + 1));
        tx[0] = max(i, 0);
        tx[1] = min(i + 1, p.r1 - 1);
        ty[0] = max(j, 0);
        ty[1] = min(j + 1, p.r1 - 1);
    };
    // ---- t2 fetch, one tile ahead: half 0 the four fp16 G0 cells (4 x C0 halves) and the raw
    // reference texel, half 1 the four fp16 G1 cells (4 x C1 halves); one register array
    // serves both halves
    constexpr int NVW = 2 * (C0 > C1 ? C0 : C1);  // 32-bit words: 4 cells x C/2
    constexpr int NRW = ((CT ? CT : 16) * 2 + 2 + 3) / 4;  // reference window words (<= 9)
    struct Fetch {
        Texel t;
        uint32_t v[NVW];   // h = 0: G0 taps (tap-major, 2 C0 words); h = 1: G1 taps (2 C1 words)
        // h = 0: the reference texel's c fp16 values as raw 32-bit words of the aligned window
        // around them, shifted into channel pairs only at the loss (loads stay in flight)
        uint32_t ref[NRW];
        uint32_t rsh;      // 16 when the texel starts 2 bytes into a word, else 0
    };
    // one fp16 cell of C channels (C/2 words) with the widest aligned vector loads
    auto load_cell_h = [&](const __half* cell, int C, uint32_t* out) {
        if (C % 8 == 0) {
            for (int e = 0; e < C / 8; ++e) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(cell) + e);
                out[4 * e] = v.x;
                out[4 * e + 1] = v.y;
                out[4 * e + 2] = v.z;
                out[4 * e + 3] = v.w;
            }
        } else if (C % 4 == 0) {
            for (int e = 0; e < C / 4; ++e) {
                const uint2 v = __ldg(reinterpret_cast<const uint2*>(cell) + e);
                out[2 * e] = v.x;
                out[2 * e + 1] = v.y;
            }
        } else {
            for (int e = 0; e < C / 2; ++e) out[e] = __ldg(reinterpret_cast<const uint32_t*>(cell) + e);
        }
    };
    auto fetch = [&](int tile, Fetch& f) {
        f.t = texel_of(tile);
        if (h == 0) {
            int tx[2], ty[2];
            taps_g0(f.t, tx, ty);
            const __half* g0 = p.noisy + p.off0;
#pragma unroll
            for (int t = 0; t < 4; ++t) load_cell_h(g0 + (ty[t >> 1] * p.r0 + tx[t & 1]) * C0, C0, f.v + t * (C0 / 2));
            const uint16_t* rp = p.ref + (int64_t)f.t.y * p.ref_stride + (int64_t)f.t.x * c;
            // the texel's 2c bytes as aligned words: full 32-bit words while they end inside the
            // texel, the last half word as a 16-bit load (no byte past the texel is read)
            const uint32_t sh = (uint32_t)(reinterpret_cast<uintptr_t>(rp) & 2u);
            const uint32_t* wp = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(rp) & ~uintptr_t(3));
            const int nb = 2 * c + (int)sh;  // window bytes
#pragma unroll
            for (int k = 0; k < NRW; ++k) {
                uint32_t v = 0u;
                if (4 * k + 4 <= nb) v = __ldg(wp + k);
                else if (4 * k + 2 == nb) v = __ldg(reinterpret_cast<const uint16_t*>(wp + k));
                f.ref[k] = v;
            }
            f.rsh = sh * 8u;
        } else {
            int tx[2], ty[2];
            uint32_t ax, ay;
            taps_g1(f.t, tx, ty, ax, ay);
            const __half* g1 = p.noisy + p.off1;
#pragma unroll
            for (int t = 0; t < 4; ++t) load_cell_h(g1 + (ty[t >> 1] * p.r1 + tx[t & 1]) * C1, C1, f.v + t * (C1 / 2));
        }
    };

    int tile = blockIdx.x * SLOTS + slot;
    const int tstride = gridDim.x * SLOTS;
    Fetch F;
    // Slot desynchronisation: both slots run the same phase sequence, so started together they
    // would stay phase-locked -- both waiting for MMAs at the same time, then competing for
    // issue slots in their epilogues.  Slot 1 starts its first tile only when slot 0 passes
    // phase TRAIN_DESYNC of its first tile (a named barrier: slot 1 sleeps, no issue slots).
    constexpr int DESYNC = SLOTS == 2 ? TRAIN_DESYNC : 0;
    if (DESYNC && slot == 1) named_bar_sync(3, 512);
    if (DESYNC && slot == 0 && tile >= p.n_tiles) named_bar_arrive(3, 512);  // no first tile
    if (tile < p.n_tiles) fetch(tile, F);
    if (issuer) mbar_wait(s_wbar, 0);  // the weight images have landed (async proxy -> MMA reads)
    int iter = 0;
    for (; tile < p.n_tiles; tile += tstride, ++iter) {
        NTC_TRACE(0);
        const Texel T = F.t;
        const bool valid = T.valid;
        uint32_t rawref[8];  // channel pairs (2o, 2o + 1) of the reference texel
#pragma unroll
        for (int o = 0; o < 8; ++o)
            rawref[o] = o < NRW ? __funnelshift_r(F.ref[o], o + 1 < NRW ? F.ref[o + 1] : 0u, F.rsh) : 0u;
        // ---- a2-a4: this half's part of the X row (canonical order, R4) -> SW128 tile(s): half 0
        // the G0 words [0, 2 C0), half 1 the G1 bilinear, PE, LOD + bias one and the padding up
        // to K1; both parts start on a 16-byte chunk (2 C0 is a multiple of 4 words)
        {
            constexpr int W0 = 2 * C0, W1N = K1 / 2 - 2 * C0;  // words of half 0 / half 1
            auto wait_pending = [&]() {
                if (pending_w) {  // the previous tile's weight-gradient MMAs still read the tiles
                    mbar_wait(bar2, phase2);
                    phase2 ^= 1;
                    tc_fence_after();
                    pending_w = false;
                }
            };
            if (h == 0) {  // G0 taps: the fp16 noisy latents are X, stored straight from the fetch
                wait_pending();
#pragma unroll
                for (int ch = 0; ch < W0 / 4; ++ch)
                    sts_row_chunk(tX + (uint32_t)(ch >> 3) * S::TILE, row, ch & 7, F.v[4 * ch], F.v[4 * ch + 1],
                                  F.v[4 * ch + 2], F.v[4 * ch + 3]);
            } else {       // G1 bilinear in fp32 from the fp16 taps, rounded once; PE; LOD
                uint32_t xw[W1N];
                int tx[2], ty[2];
                uint32_t ax, ay;
                taps_g1(T, tx, ty, ax, ay);
                const uint32_t wq[4] = {(16u - ax) * (16u - ay), ax * (16u - ay), (16u - ax) * ay, ax * ay};
                if constexpr (TRAIN_G1_H2) {
                    // packed fp16 bilinear: the weights (multiples of 1/256) are exact in fp16, each
                    // HFMA2 step rounds once
                    __half2 acc2[C1 / 2];
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const __half2 w2 = __float2half2_rn((float)wq[t] * (1.0f / 256.0f));
#pragma unroll
                        for (int e = 0; e < C1 / 2; ++e) {
                            const __half2 a2 = *reinterpret_cast<const __half2*>(&F.v[t * (C1 / 2) + e]);
                            acc2[e] = t == 0 ? __hmul2(a2, w2) : __hfma2(a2, w2, acc2[e]);
                        }
                    }
#pragma unroll
                    for (int e = 0; e < C1 / 2; ++e) xw[e] = *reinterpret_cast<const uint32_t*>(&acc2[e]);
                } else {
                float acc[C1];
#pragma unroll
                for (int e = 0; e < C1; ++e) acc[e] = 0.0f;
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float wf = (float)wq[t] * (1.0f / 256.0f);
#pragma unroll
                    for (int e = 0; e < C1 / 2; ++e) {
                        const float2 a2 = __half22float2(*reinterpret_cast<const __half2*>(&F.v[t * (C1 / 2) + e]));
                        acc[2 * e + 0] = fmaf(wf, a2.x, acc[2 * e + 0]);
                        acc[2 * e + 1] = fmaf(wf, a2.y, acc[2 * e + 1]);
                    }
                }
#pragma unroll
                for (int e = 0; e < C1; e += 2) xw[e / 2] = h2u(acc[e], acc[e + 1]);
                }
                constexpr int PEW = C1 / 2;  // word index inside this half
                xw[PEW + 0] = s_pe[4 * (T.x & 7) + 0];
                xw[PEW + 1] = s_pe[4 * (T.x & 7) + 1];
                xw[PEW + 2] = s_pe[4 * (T.x & 7) + 2];
                xw[PEW + 3] = s_pe[4 * (T.y & 7) + 0];
                xw[PEW + 4] = s_pe[4 * (T.y & 7) + 1];
                xw[PEW + 5] = s_pe[4 * (T.y & 7) + 2];
                xw[PEW + 6] = p.lod_word;
#pragma unroll
                for (int e = PEW + 7; e < W1N; ++e) xw[e] = 0u;
                wait_pending();
#pragma unroll
                for (int ch = 0; ch < W1N / 4; ++ch) {
                    const int g = W0 / 4 + ch;  // chunk of the K1-wide row: atom g / 8, chunk g % 8
                    sts_row_chunk(tX + (uint32_t)(g >> 3) * S::TILE, row, g & 7, xw[4 * ch], xw[4 * ch + 1],
                                  xw[4 * ch + 2], xw[4 * ch + 3]);
                }
            }
        }
        NTC_TRACE(17);
        sync_slot();
        NTC_TRACE(1);
        // ---- t3: forward.  Z1 = X W1^T (+b1)
        if (issuer) {
            tc_fence_after();
            if constexpr (CH && KA == 1) {
                mma_chain4_commit_warp<2, 2>(t_s, dX, dW1, ID64, 0, bar);
            } else if constexpr (CH) {  // K1 = 80 / 96: atom 0's chain, then atom 1's one or two steps
                mma_chain4_warp<2, 2>(t_s, dX, dW1, ID64, 0);
                constexpr uint64_t A1 = S::TILE >> 4, B1 = 8192 >> 4;
                if constexpr (K1 / 16 == 6) mma_f16_ss_warp(t_s, dX + A1, dW1 + B1, ID64, 1);
                mma1_commit_warp(t_s, dX + A1 + (K1 / 16 == 6 ? 2 : 0), dW1 + B1 + (K1 / 16 == 6 ? 2 : 0), ID64, 1, bar);
            } else {
#pragma unroll
                for (int kk = 0; kk < K1 / 16; ++kk)
                    mma(t_s, dX + (uint64_t)(((kk >> 2) * S::TILE + (kk & 3) * 32) >> 4),
                        dW1 + (uint64_t)(((kk >> 2) * 8192 + (kk & 3) * 32) >> 4), ID64, kk > 0);
                commit(bar);
            }
        }
        if (tile + tstride < p.n_tiles) fetch(tile + tstride, F);  // next tile's loads in flight
        wait_mma();
        NTC_TRACE(2);
        // two 16-column tcgen05.ld per half, the second in flight while the first is processed
        // (the register-dependent wait orders the uses after it)
        auto hidden_epilogue = [&](uint32_t tH, uint32_t tG) {
            uint32_t r[2][16];
            tmem_ld16(t_s + lane_off + 32 * h, r[0]);
            tmem_wait_ld_r16(r[0]);
            tmem_ld16(t_s + lane_off + 32 * h + 16, r[1]);
#pragma unroll
            for (int part = 0; part < 2; ++part) {
                if (part == 1) tmem_wait_ld_r16(r[1]);
                uint32_t hv[8], gv[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float z0 = __uint_as_float(r[part][2 * i]), z1 = __uint_as_float(r[part][2 * i + 1]);
                    if constexpr (ACT == 0) {
                        hgelu_and_grad2(z0, z1, hv[i], gv[i]);
                    } else {
                        float h0, h1, g0, g1;
                        act_and_grad<ACT>(z0, h0, g0);
                        act_and_grad<ACT>(z1, h1, g1);
                        hv[i] = h2u(h0, h1);
                        gv[i] = h2u(g0, g1);
                    }
                }
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {
                    const int ch = 4 * h + 2 * part + cc;
                    sts_row_chunk(tH, row, ch, hv[4 * cc], hv[4 * cc + 1], hv[4 * cc + 2], hv[4 * cc + 3]);
                    sts_row_chunk(tG, row, ch, gv[4 * cc], gv[4 * cc + 1], gv[4 * cc + 2], gv[4 * cc + 3]);
                }
            }
        };
        hidden_epilogue(tH1, tG1);
        NTC_TRACE(19);
        sync_slot();
        NTC_TRACE(3);
        if (DESYNC == 3 && slot == 0 && iter == 0) named_bar_arrive(3, 512);
        // Z2 = H1 W2^T + b2
        if (issuer) {
            tc_fence_after();
            if constexpr (CH) {
                mma_chain4_warp<2, 2>(t_s, dH1, dW2, ID64, 0);
                mma1_commit_warp(t_s, dONES, dB2, ID64, 1, bar);
            } else {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) mma(t_s, dH1 + 2 * kk, dW2 + 2 * kk, ID64, kk > 0);
                mma(t_s, dONES, dB2, ID64, 1);
                commit(bar);
            }
        }
        wait_mma();
        NTC_TRACE(4);
        hidden_epilogue(tH2, tG2);
        if constexpr (HM == 2) {  // Z3 = H2 W2b^T + b2b
            sync_slot();
            if (issuer) {
                tc_fence_after();
                if constexpr (CH) {
                    mma_chain4_warp<2, 2>(t_s, dH2, dW2B, ID64, 0);
                    mma1_commit_warp(t_s, dONES, dB2B, ID64, 1, bar);
                } else {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) mma(t_s, dH2 + 2 * kk, dW2B + 2 * kk, ID64, kk > 0);
                    mma(t_s, dONES, dB2B, ID64, 1);
                    commit(bar);
                }
            }
            wait_mma();
            hidden_epilogue(tH3, tG3);
        }
        NTC_TRACE(21);
        sync_slot();
        NTC_TRACE(5);
        if (DESYNC == 5 && slot == 0 && iter == 0) named_bar_arrive(3, 512);
        // Y = H_last W3^T + b3
        if (issuer) {
            tc_fence_after();
            if constexpr (CH) {
                mma_chain4_warp<2, 2>(t_s, dHL, dW3, ID16, 0);
                mma1_commit_warp(t_s, dONES, dB3, ID16, 1, bar);
            } else {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) mma(t_s, dHL + 2 * kk, dW3 + 2 * kk, ID16, kk > 0);
                mma(t_s, dONES, dB3, ID16, 1);
                commit(bar);
            }
        }
        wait_mma();
        NTC_TRACE(6);
        // ---- t4: mean-L2 loss (R17) on half 0 (it holds the reference); delta3 = 2 (y - R)
        // fed unscaled, 1/(B c) applied in fp32
        if (h == 0) {
            uint32_t r[16];
            tmem_ld16(t_s + lane_off, r);
            tmem_wait_ld();
            float d3[16];
#pragma unroll
            for (int o = 0; o < 16; ++o) {
                const float rf = __half2float(__ushort_as_half((uint16_t)(rawref[o >> 1] >> (16 * (o & 1)))));
                const float e = (valid && o < c) ? __uint_as_float(r[o]) - rf : 0.0f;
                loss_acc = fmaf(e, e, loss_acc);
                d3[o] = 2.0f * e;
            }
            sts_row_chunk(tD3, row, 0, h2u(d3[0], d3[1]), h2u(d3[2], d3[3]), h2u(d3[4], d3[5]), h2u(d3[6], d3[7]));
            sts_row_chunk(tD3, row, 1, h2u(d3[8], d3[9]), h2u(d3[10], d3[11]), h2u(d3[12], d3[13]),
                          h2u(d3[14], d3[15]));
        }
        NTC_TRACE(23);
        sync_slot();
        NTC_TRACE(7);
        if (DESYNC == 7 && slot == 0 && iter == 0) named_bar_arrive(3, 512);
        // ---- t5: dH_last = d3 W3
        if (issuer) {
            tc_fence_after();
            if constexpr (CH) {
                mma1_commit_warp(t_s, dD3, mW3, ID64_BT, 0, bar);
            } else {
                mma(t_s, dD3, mW3, ID64_BT, 0);
                commit(bar);
            }
            if (TRAIN_DWB_EARLY && CH) {
                mma_chain8_warp<128, 128>(t_acc_b, mXHL, mD3, ID16_AB, !first);
            } else if (TRAIN_DWB_EARLY) {  // dW3/db3 += [X^T; H_last^T] delta3: its operands are final here
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma(t_acc_b, mXHL + (uint64_t)(kk * 128), mD3 + (uint64_t)(kk * 128), ID16_AB,
                               (!first || kk > 0) ? 1u : 0u);
            }
        }
        wait_mma();
        NTC_TRACE(8);
        auto delta_epilogue = [&](uint32_t tG) {  // delta = fp16(dH) * hardGELU'(Z), in place
            if constexpr (BF16ACC) {  // dH already fp16: two packed 16-column loads per half
                uint32_t r[2][8];
                tmem_ld8_pack(t_s + lane_off + 32 * h, r[0]);
                tmem_wait_ld_r8(r[0]);
                tmem_ld8_pack(t_s + lane_off + 32 * h + 16, r[1]);
#pragma unroll
                for (int part = 0; part < 2; ++part) {
                    if (part == 1) tmem_wait_ld_r8(r[1]);
#pragma unroll
                    for (int cc = 0; cc < 2; ++cc) {
                        const int ch = 4 * h + 2 * part + cc;
                        const uint4 gq = lds_row_chunk(tG, row, ch);
                        const uint32_t gw[4] = {gq.x, gq.y, gq.z, gq.w};
                        uint32_t o[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const __half2 dv = __hmul2(*reinterpret_cast<const __half2*>(&r[part][4 * cc + e]),
                                                       *reinterpret_cast<const __half2*>(&gw[e]));
                            o[e] = *reinterpret_cast<const uint32_t*>(&dv);
                        }
                        sts_row_chunk(tG, row, ch, o[0], o[1], o[2], o[3]);
                    }
                }
                return;
            }
            uint32_t r[2][16];
            tmem_ld16(t_s + lane_off + 32 * h, r[0]);
            tmem_wait_ld_r16(r[0]);
            tmem_ld16(t_s + lane_off + 32 * h + 16, r[1]);
#pragma unroll
            for (int part = 0; part < 2; ++part) {
                if (part == 1) tmem_wait_ld_r16(r[1]);
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {
                    const int ch = 4 * h + 2 * part + cc;
                    const uint4 gq = lds_row_chunk(tG, row, ch);
                    const uint32_t gw[4] = {gq.x, gq.y, gq.z, gq.w};
                    uint32_t o[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const __half2 g2 = *reinterpret_cast<const __half2*>(&gw[e]);
                        const int col = 8 * cc + 2 * e;
                        const uint32_t aw = h2u(__uint_as_float(r[part][col]), __uint_as_float(r[part][col + 1]));
                        const __half2 dv = __hmul2(*reinterpret_cast<const __half2*>(&aw), g2);
                        o[e] = *reinterpret_cast<const uint32_t*>(&dv);
                    }
                    sts_row_chunk(tG, row, ch, o[0], o[1], o[2], o[3]);
                }
            }
        };
        delta_epilogue(tGL);  // the last G tile now holds its delta
        if constexpr (HM == 2) {  // dH2 = d3h W2b ; delta2
            sync_slot();
            if (issuer) {
                tc_fence_after();
                if constexpr (CH) {
                    mma_chain4_commit_warp<2, 128>(t_s, dG3, mW2B, ID64_BT, 0, bar);
                } else {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        mma(t_s, dG3 + 2 * kk, mW2B + (uint64_t)(kk * 128), ID64_BT, kk > 0);
                    commit(bar);
                }
            }
            wait_mma();
            delta_epilogue(tG2);
        }
        NTC_TRACE(25);
        sync_slot();
        NTC_TRACE(9);
        // dH1 = d2 W2
        if (issuer) {
            tc_fence_after();
            if constexpr (CH) {
                mma_chain4_commit_warp<2, 128>(t_s, dG2, mW2, ID64_BT, 0, bar);
            } else {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) mma(t_s, dG2 + 2 * kk, mW2 + (uint64_t)(kk * 128), ID64_BT, kk > 0);
                commit(bar);
            }
        }
        wait_mma();
        NTC_TRACE(10);
        delta_epilogue(tG1);  // G1 tile now holds delta1
        NTC_TRACE(27);
        sync_slot();
        NTC_TRACE(11);
        // dX = d1 W1 (latent columns) ; weight gradients accumulated in TMEM
        if (issuer && CH) {  // the same groups, one asm block each
            tc_fence_after();
            mma_chain4_commit_warp<2, 128>(t_s, dG1, mW1, IDX_BT, 0, bar);
            if (!TRAIN_DWB_EARLY) mma_chain8_warp<128, 128>(t_acc_b, mXHL, mD3, ID16_AB, !first);
            if constexpr (HM == 2) mma_chain8_warp<128, 128>(t_acc_m, mXH2, mG3, ID64_AB, !first);
            if constexpr (KA == 1) {
                mma_chain8_commit_warp<128, 128>(t_acc_a, mXH1, mG1, ID128_AB, !first, bar2);
            } else {
                mma_chain8_warp<128, 128>(t_acc_a + 64, mXH1, mG2, ID64_AB, !first);
                mma_chain8_commit_warp<128, 128>(t_acc_a, mXX, mG1, ID64_AB, !first, bar2);
            }
        } else if (issuer) {
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                mma(t_s, dG1 + 2 * kk, mW1 + (uint64_t)(kk * 128), IDX_BT, kk > 0);
            commit(bar);
            // weight gradients, off the critical path: they run while this tile scatters and
            // the next tile fetches; bar2 is waited before the next tile overwrites the tiles
            if (!TRAIN_DWB_EARLY) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma(t_acc_b, mXHL + (uint64_t)(kk * 128), mD3 + (uint64_t)(kk * 128), ID16_AB,
                               (!first || kk > 0) ? 1u : 0u);
            }
            if constexpr (HM == 2) {  // dW2b/db2b += [X^T; H2^T] delta3h
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma(t_acc_m, mXH2 + (uint64_t)(kk * 128), mG3 + (uint64_t)(kk * 128), ID64_AB,
                               (!first || kk > 0) ? 1u : 0u);
            }
            if constexpr (KA == 1) {
                // dW1/db1 and dW2/db2 in one N = 128 MMA per K step: [X^T; H1^T] [delta1 | delta2]
                // (adjacent tiles; the diagonal blocks are used, rows 64-127 of the delta1 half
                // and rows < 64 of the delta2 half except the constant row are not)
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma(t_acc_a, mXH1 + (uint64_t)(kk * 128), mG1 + (uint64_t)(kk * 128), ID128_AB,
                               (!first || kk > 0) ? 1u : 0u);
            } else {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma(t_acc_a + 64, mXH1 + (uint64_t)(kk * 128), mG2 + (uint64_t)(kk * 128), ID64_AB,
                               (!first || kk > 0) ? 1u : 0u);
                // dW1/db1: [X0^T; X1^T] delta1
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma(t_acc_a, mXX + (uint64_t)(kk * 128), mG1 + (uint64_t)(kk * 128), ID64_AB,
                               (!first || kk > 0) ? 1u : 0u);
            }
            commit(bar2);
        }
        wait_mma();
        NTC_TRACE(12);
        first = false;
        pending_w = true;
        // ---- t7: latent-gradient scatter: half 0 the G0 taps (unweighted), half 1 the G1 taps
        // (bilinear-weighted).  Neighbouring texels share tap cells (runs of 4 texels share all
        // four G0 cells and runs of 8 share the G1 cells at LOD 0), so each run is summed to its
        // first lane with two (G0) / three (G1) shuffle steps and only run heads issue the
        // vector reductions -- no global contention storm.
        if constexpr (BF16ACC) {
            // dX is fp16 in TMEM: the run sums run on packed half2 words (channel pairs), then
            // widen to fp32 for the scaled vector reductions (the fp16 run sums of <= 4 / 8 texels
            // add one rounding, far inside the gradient tolerance R21)
            const float s = p.inv_bc;
            const bool on = valid && !p.freeze;
            if (h == 0) {
                constexpr int NW0 = 2 * C0;  // words of the 4 x C0 G0 values (tap-major)
                uint32_t g0w[NW0];
#pragma unroll
                for (int w = 0; w + 16 <= NW0; w += 16) {
                    uint32_t q[16];
                    tmem_ld16_pack(t_s + lane_off + 2 * w, q);
                    tmem_wait_ld_r16(q);
#pragma unroll
                    for (int e = 0; e < 16; ++e) g0w[w + e] = on ? q[e] : 0u;
                }
                if constexpr (NW0 % 16 == 8) {
                    uint32_t q[8];
                    tmem_ld8_pack(t_s + lane_off + 2 * (NW0 - 8), q);
                    tmem_wait_ld_r8(q);
#pragma unroll
                    for (int e = 0; e < 8; ++e) g0w[NW0 - 8 + e] = on ? q[e] : 0u;
                }
                int tx0[2], ty0[2];
                taps_g0(T, tx0, ty0);
                float* gl0 = p.grad_lat + p.off0;
                const uint32_t kx0 = on ? (uint32_t)(tx0[0] | (tx0[1] << 16)) : 0xFFFFFFF0u - lane;
                const uint32_t ky0 = (uint32_t)(ty0[0] | (ty0[1] << 16));
#pragma unroll
                for (int d = 1; d <= 2; d <<= 1) {
                    const uint32_t nx0 = __shfl_down_sync(0xffffffffu, kx0, d);
                    const uint32_t ny0 = __shfl_down_sync(0xffffffffu, ky0, d);
                    const bool s0 = lane + d < 32 && nx0 == kx0 && ny0 == ky0;
#pragma unroll
                    for (int i = 0; i < NW0; ++i) {
                        const uint32_t o = __shfl_down_sync(0xffffffffu, g0w[i], d);
                        const __half2 sum = __hadd2(*reinterpret_cast<const __half2*>(&g0w[i]),
                                                    *reinterpret_cast<const __half2*>(&o));
                        if (s0) g0w[i] = *reinterpret_cast<const uint32_t*>(&sum);
                    }
                }
                const uint32_t px0 = __shfl_up_sync(0xffffffffu, kx0, 1), py0 = __shfl_up_sync(0xffffffffu, ky0, 1);
                if (on && (lane == 0 || px0 != kx0 || py0 != ky0)) {
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        float* dst = gl0 + ((int64_t)ty0[t >> 1] * p.r0 + tx0[t & 1]) * C0;
#pragma unroll
                        for (int e = 0; e < C0; e += 4) {
                            const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&g0w[(t * C0 + e) / 2]));
                            const float2 b =
                                __half22float2(*reinterpret_cast<const __half2*>(&g0w[(t * C0 + e) / 2 + 1]));
                            red_add_v4(dst + e, s * a.x, s * a.y, s * b.x, s * b.y);
                        }
                    }
                }
            } else {
                constexpr int NW1 = C1 / 2;
                constexpr int NQ = NW1 <= 8 ? 8 : 16;
                uint32_t q[NQ];
                if constexpr (NQ == 8) {
                    tmem_ld8_pack(t_s + lane_off + 4 * C0, *reinterpret_cast<uint32_t(*)[8]>(q));
                    tmem_wait_ld_r8(*reinterpret_cast<uint32_t(*)[8]>(q));
                } else {
                    tmem_ld16_pack(t_s + lane_off + 4 * C0, *reinterpret_cast<uint32_t(*)[16]>(q));
                    tmem_wait_ld_r16(*reinterpret_cast<uint32_t(*)[16]>(q));
                }
                int tx1[2], ty1[2];
                uint32_t axq, ayq;
                taps_g1(T, tx1, ty1, axq, ayq);
                float* gl1 = p.grad_lat + p.off1;
                const uint32_t kx1 = on ? (uint32_t)(tx1[0] | (tx1[1] << 16)) : 0xFFFFFFF0u - lane;
                const uint32_t ky1 = (uint32_t)T.y;
                const uint32_t ky1b = (uint32_t)(ty1[0] | (ty1[1] << 16));
                // x-weights (multiples of 1/16, exact in fp16) applied per texel, y-weights at the head
                const float ax = (float)axq * (1.0f / 16.0f);
                const float ay = (float)ayq * (1.0f / 16.0f);
                const __half2 wa = __float2half2_rn(1.0f - ax), wb = __float2half2_rn(ax);
                uint32_t g1w[2 * NW1];
#pragma unroll
                for (int e = 0; e < NW1; ++e) {
                    const __half2 v = *reinterpret_cast<const __half2*>(&q[e]);
                    const __half2 va = __hmul2(v, wa), vb = __hmul2(v, wb);
                    g1w[e] = on ? *reinterpret_cast<const uint32_t*>(&va) : 0u;
                    g1w[NW1 + e] = on ? *reinterpret_cast<const uint32_t*>(&vb) : 0u;
                }
#pragma unroll
                for (int d = 1; d <= 4; d <<= 1) {
                    const uint32_t nx1 = __shfl_down_sync(0xffffffffu, kx1, d);
                    const uint32_t ny1 = __shfl_down_sync(0xffffffffu, ky1, d);
                    const uint32_t ny1b = __shfl_down_sync(0xffffffffu, ky1b, d);
                    const bool s1 = lane + d < 32 && nx1 == kx1 && ny1 == ky1 && ny1b == ky1b;
#pragma unroll
                    for (int i = 0; i < 2 * NW1; ++i) {
                        const uint32_t o = __shfl_down_sync(0xffffffffu, g1w[i], d);
                        const __half2 sum = __hadd2(*reinterpret_cast<const __half2*>(&g1w[i]),
                                                    *reinterpret_cast<const __half2*>(&o));
                        if (s1) g1w[i] = *reinterpret_cast<const uint32_t*>(&sum);
                    }
                }
                const uint32_t px1 = __shfl_up_sync(0xffffffffu, kx1, 1), py1 = __shfl_up_sync(0xffffffffu, ky1, 1);
                const uint32_t py1b = __shfl_up_sync(0xffffffffu, ky1b, 1);
                if (on && (lane == 0 || px1 != kx1 || py1 != ky1 || py1b != ky1b)) {
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const float wy = (t >> 1) ? ay : 1.0f - ay;
                        const uint32_t* Sv = g1w + (t & 1) * NW1;
                        float* dst = gl1 + ((int64_t)ty1[t >> 1] * p.r1 + tx1[t & 1]) * C1;
                        const float sw = s * wy;
                        if (sw != 0.0f) {
                            if constexpr (C1 % 4 == 0) {
#pragma unroll
                                for (int e = 0; e < C1; e += 4) {
                                    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&Sv[e / 2]));
                                    const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&Sv[e / 2 + 1]));
                                    red_add_v4(dst + e, sw * a.x, sw * a.y, sw * b.x, sw * b.y);
                                }
                            } else {
#pragma unroll
                                for (int e = 0; e < C1; e += 2) {
                                    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&Sv[e / 2]));
                                    red_add_v2(dst + e, sw * a.x, sw * a.y);
                                }
                            }
                        }
                    }
                }
            }
        } else {
            const float s = p.inv_bc;
            const bool on = valid && !p.freeze;
            if (h == 0) {
                uint32_t r[4 * C0];
#pragma unroll
                for (int blk = 0; blk < C0 / 4; ++blk) {
                    uint32_t q16[16];
                    tmem_ld16(t_s + lane_off + 16 * blk, q16);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 16; ++e) r[16 * blk + e] = q16[e];
                }
                int tx0[2], ty0[2];
                taps_g0(T, tx0, ty0);
                float* gl0 = p.grad_lat + p.off0;
                const uint32_t kx0 = on ? (uint32_t)(tx0[0] | (tx0[1] << 16)) : 0xFFFFFFF0u - lane;
                const uint32_t ky0 = (uint32_t)(ty0[0] | (ty0[1] << 16));
                float g0v[4 * C0];
#pragma unroll
                for (int i = 0; i < 4 * C0; ++i) g0v[i] = on ? __uint_as_float(r[i]) : 0.0f;
#pragma unroll
                for (int d = 1; d <= 2; d <<= 1) {
                    const uint32_t nx0 = __shfl_down_sync(0xffffffffu, kx0, d);
                    const uint32_t ny0 = __shfl_down_sync(0xffffffffu, ky0, d);
                    const bool s0 = lane + d < 32 && nx0 == kx0 && ny0 == ky0;
#pragma unroll
                    for (int i = 0; i < 4 * C0; ++i) {
                        const float o = __shfl_down_sync(0xffffffffu, g0v[i], d);
                        if (s0) g0v[i] += o;
                    }
                }
                const uint32_t px0 = __shfl_up_sync(0xffffffffu, kx0, 1), py0 = __shfl_up_sync(0xffffffffu, ky0, 1);
                // runs never exceed 4 lanes (r0 / w_m >= 1/4 for the compiled profiles)
                if (on && (lane == 0 || px0 != kx0 || py0 != ky0)) {
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        float* dst = gl0 + ((int64_t)ty0[t >> 1] * p.r0 + tx0[t & 1]) * C0;
#pragma unroll
                        for (int e = 0; e < C0; e += 4)
                            red_add_v4(dst + e, s * g0v[t * C0 + e], s * g0v[t * C0 + e + 1], s * g0v[t * C0 + e + 2],
                                       s * g0v[t * C0 + e + 3]);
                    }
                }
            } else {
                constexpr int NR = C1 <= 16 ? 16 : 32;
                uint32_t r[NR];
                if constexpr (NR == 16)
                    tmem_ld16(t_s + lane_off + 4 * C0, r);
                else
                    tmem_ld32(t_s + lane_off + 4 * C0, r);
                tmem_wait_ld();
                int tx1[2], ty1[2];
                uint32_t axq, ayq;
                taps_g1(T, tx1, ty1, axq, ayq);
                float* gl1 = p.grad_lat + p.off1;
                const uint32_t kx1 = on ? (uint32_t)(tx1[0] | (tx1[1] << 16)) : 0xFFFFFFF0u - lane;
                const uint32_t ky1 = (uint32_t)T.y;  // same y => same y-weights within a G1 run
                const uint32_t ky1b = (uint32_t)(ty1[0] | (ty1[1] << 16));
                // per x-tap a, S_a = sum over the run of wx_a * dX_G1 (wy is constant in a run)
                const float ax = (float)axq * (1.0f / 16.0f);  // x-weight of tap column 1
                const float ay = (float)ayq * (1.0f / 16.0f);  // y-weight of tap row 1
                float g1v[2 * C1];
#pragma unroll
                for (int e = 0; e < C1; ++e) {
                    const float v = on ? __uint_as_float(r[e]) : 0.0f;
                    g1v[e] = (1.0f - ax) * v;
                    g1v[C1 + e] = ax * v;
                }
#pragma unroll
                for (int d = 1; d <= 4; d <<= 1) {
                    const uint32_t nx1 = __shfl_down_sync(0xffffffffu, kx1, d);
                    const uint32_t ny1 = __shfl_down_sync(0xffffffffu, ky1, d);
                    const uint32_t ny1b = __shfl_down_sync(0xffffffffu, ky1b, d);
                    const bool s1 = lane + d < 32 && nx1 == kx1 && ny1 == ky1 && ny1b == ky1b;
#pragma unroll
                    for (int i = 0; i < 2 * C1; ++i) {
                        const float o = __shfl_down_sync(0xffffffffu, g1v[i], d);
                        if (s1) g1v[i] += o;
                    }
                }
                const uint32_t px1 = __shfl_up_sync(0xffffffffu, kx1, 1), py1 = __shfl_up_sync(0xffffffffu, ky1, 1);
                const uint32_t py1b = __shfl_up_sync(0xffffffffu, ky1b, 1);
                // runs never exceed 8 lanes (r1 / w_m >= 1/8)
                if (on && (lane == 0 || px1 != kx1 || py1 != ky1 || py1b != ky1b)) {
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const float wy = (t >> 1) ? ay : 1.0f - ay;
                        const float* Sv = g1v + (t & 1) * C1;
                        float* dst = gl1 + ((int64_t)ty1[t >> 1] * p.r1 + tx1[t & 1]) * C1;
                        const float sw = s * wy;
                        if (sw != 0.0f) {
                            if constexpr (C1 % 4 == 0) {
#pragma unroll
                                for (int e = 0; e < C1; e += 4)
                                    red_add_v4(dst + e, sw * Sv[e], sw * Sv[e + 1], sw * Sv[e + 2], sw * Sv[e + 3]);
                            } else {  // 8-byte aligned cells (C1 = 10)
#pragma unroll
                                for (int e = 0; e < C1; e += 2) red_add_v2(dst + e, sw * Sv[e], sw * Sv[e + 1]);
                            }
                        }
                    }
                }
            }
        }
        NTC_TRACE(15);
        tc_fence_before();
    }

    NTC_TRACE_K(2, (uint32_t)clock64());
    pdl_launch_dependents();  // the reduce / Adam kernel may launch as CTAs retire
    if (pending_w) {
        mbar_wait(bar2, phase2);
        phase2 ^= 1;
        tc_fence_after();
    }
    NTC_TRACE_K(6, (uint32_t)clock64());
    // ---- t6: the CTA's weight-gradient partial (unscaled, one per CTA, fixed order).  Each
    // slot writes its TMEM accumulators into its own (now idle) tile area in ABI order -- every
    // accumulator (row, column) used maps to one ABI index, and consecutive rows (lanes) to
    // consecutive addresses -- then all threads add the slots' buffers and store the partial
    // with coalesced 16-byte stores.  Half 0 handles the dW1/db1 columns [0, 64) (and the
    // middle layer's dW2b/db2b at depth 2), half 1 the dW2/db2 columns [64, 128) and dW3/db3.
    {
        const bool have = !first;  // a slot without tiles never wrote its accumulators
        const int m = row;         // stacked rows: X features (64 per atom), then H units at [64,128)
        const int P1 = D * HID, o2 = P1 + HID, o2b = o2 + HID * HID + HID, o3 = P1 + HID + HM * (HID * HID + HID);
        float* buf = reinterpret_cast<float*>(smem + S::WEND + (uint32_t)slot * S::WG_BYTES);
        // 64 accumulator columns at t -> buf[base + col * stride] (base < 0: row unused)
        auto put64 = [&](uint32_t t, int base, int stride) {
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) {
                uint32_t r[32];
                tmem_ld32(t + lane_off + 32 * blk, r);
                tmem_wait_ld();
                if (base >= 0) {
#pragma unroll
                    for (int e = 0; e < 32; ++e) buf[base + (32 * blk + e) * stride] = have ? __uint_as_float(r[e]) : 0.0f;
                }
            }
        };
        sync_slot();  // the slot's tiles are free (its last weight-gradient MMAs were waited above)
        if (h == 0) {
            put64(t_acc_a, m < D ? m : (m == D ? P1 : -1), m < D ? D : 1);  // dW1[j][i], db1[j]
            if constexpr (HM == 2)
                put64(t_acc_m, m >= 64 ? o2b + (m - 64) : (m == DX ? o2b + HID * HID : -1), m >= 64 ? HID : 1);
        } else {
            put64(t_acc_a + 64, m >= 64 ? o2 + (m - 64) : (m == DX ? o2 + HID * HID : -1), m >= 64 ? HID : 1);
            uint32_t r[16];
            tmem_ld16(t_acc_b + lane_off, r);
            tmem_wait_ld();
            const int base = m >= 64 ? o3 + (m - 64) : (m == DX ? o3 + HID * c : -1), stride = m >= 64 ? HID : 1;
            if (base >= 0) {
#pragma unroll
                for (int o = 0; o < 16; ++o)
                    if (o < c) buf[base + o * stride] = have ? __uint_as_float(r[o]) : 0.0f;  // dW3[o][i], db3[o]
            }
        }
        __syncthreads();
        const float4* b0 = reinterpret_cast<const float4*>(smem + S::WEND);
        const float4* b1 = reinterpret_cast<const float4*>(smem + S::WEND + S::WG_BYTES);
        float4* part = reinterpret_cast<float4*>(p.partial + (size_t)blockIdx.x * p.Pst);
        for (int i = tid; i < p.Pst / 4; i += blockDim.x) {
            float4 v = b0[i];
            if constexpr (SLOTS == 2) {
                const float4 u = b1[i];
                v.x += u.x;
                v.y += u.y;
                v.z += u.z;
                v.w += u.w;
            }
            part[i] = v;  // entries [P, Pst) are never read
        }
    }
    NTC_TRACE_K(10, (uint32_t)clock64());
    {
        float v = loss_acc;
#pragma unroll
        for (int sft = 16; sft > 0; sft >>= 1) v += __shfl_xor_sync(0xffffffffu, v, sft);
        if (lane == 0 && h == 0) atomicAdd(&s_loss[slot], v);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid < SLOTS) p.loss_partial[blockIdx.x * SLOTS + tid] = s_loss[tid];
    NTC_TRACE_K(3, (uint32_t)clock64());
#ifdef NTC_TRAIN_TRACE
    NTC_TRACE_K(5, gtimer_lo());
#endif
    if (warp == 0) tmem_dealloc(*s_tmem, 512);
}

constexpr int RED_MAXK = 32;  // nparts <= 8 * RED_MAXK (grid <= 256 CTAs)
struct ReduceArgs {
    const float* partial;
    size_t part_stride;
    const float* loss_partial;
    int nparts, P;
    int nloss;  // loss partials (CTAs x slots)
    float inv_bc;
    float* grad;
    float* loss;
    int32_t* status;
};

// one block: 32 parameters x 8 partial groups (blockIdx `blk`); returns the reduced, scaled
// gradient of parameter `i` on the group-0 threads (undefined elsewhere)
__device__ __forceinline__ float reduce_block(const ReduceArgs& r, int blk, int& i_out) {
    __shared__ float s[8][33];
    __shared__ float sl[256];
    const int px = threadIdx.x & 31, g = threadIdx.x >> 5;
    const int i = blk * 32 + px;
    float v[RED_MAXK];
#pragma unroll
    for (int k = 0; k < RED_MAXK; ++k) {
        const int w = g + 8 * k;
        v[k] = (i < r.P && w < r.nparts) ? __ldg(r.partial + (size_t)w * r.part_stride + i) : 0.0f;
    }
    float t = 0.0f;
#pragma unroll
    for (int k = 0; k < RED_MAXK; ++k) t += v[k];
    s[g][px] = t;
    if (blk == 0) {
        const int nl = r.nloss;  // <= 2 * 256
        float l = 0.0f;
        if ((int)threadIdx.x < nl) l = r.loss_partial[threadIdx.x];
        if ((int)threadIdx.x + 256 < nl) l += r.loss_partial[threadIdx.x + 256];
        sl[threadIdx.x] = l;
    }
    __syncthreads();
    float gr = 0.0f;
    if (g == 0 && i < r.P) {
        float u = 0.0f;
#pragma unroll
        for (int k = 0; k < 8; ++k) u += s[k][px];
        gr = u * r.inv_bc;
        r.grad[i] = gr;
    }
    if (blk == 0) {
        for (int hh = 128; hh > 0; hh >>= 1) {
            if ((int)threadIdx.x < hh) sl[threadIdx.x] += sl[threadIdx.x + hh];
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            const float l = sl[0] * r.inv_bc;
            *r.loss = l;
            if (!isfinite(l) && r.status) atomicOr(r.status, (int)NTC_ERR_NONFINITE);
        }
    }
    i_out = (g == 0 && i < r.P) ? i : -1;
    return gr;
}

// fixed-order reduction of the per-CTA partials (deterministic), scaled by 1/(B c): block =
// 32 parameters x 8 partial groups; group g owns partials g, g+8, ... and issues all of its
// (<= RED_MAXK) loads before summing them in order; the 8 group sums are then added in
// order.  Block 0 also reduces the loss partials with a fixed-shape tree.
__global__ void __launch_bounds__(256) reduce_kernel(const __grid_constant__ ReduceArgs r) {
    pdl_wait();  // the training kernel's partials are complete
    int i;
    reduce_block(r, blockIdx.x, i);
}

// ------------------------------------------------------------------ t8: Adam + clamp
struct AdamParams {
    Box box[MAX_BOXES];
    int32_t nbox;
    int32_t box_start[MAX_BOXES + 1];
    int32_t dense_latents;
    int64_t n_latents;
    int32_t P;
    float* params;
    float* m_par;
    float* v_par;
    const float* grad_par;
    float* latents;
    float* m_lat;
    float* v_lat;
    const float* grad_lat;
    float lr_w, lr_l, b1, b2, eps, c1, c2;  // c1 = 1 - b1^t, c2 = 1 - b2^t
    int32_t freeze;                         // skip the latents (frozen phase)
    // dense-latent mode: per-grid bits lookup
    int32_t ngrid;
    int64_t grid_start[2 * MAX_LEVELS + 1];
    int32_t grid_bits[2 * MAX_LEVELS];
};

__device__ __forceinline__ void adam_one(float& p, float& m, float& v, float g, float lr, const AdamParams& a) {
    m = a.b1 * m + (1.0f - a.b1) * g;
    v = a.b2 * v + (1.0f - a.b2) * g * g;
    p -= lr * (m / a.c1) / (sqrtf(v / a.c2) + a.eps);
}

__device__ __forceinline__ void adam_weight(const AdamParams& a, int64_t i, float g) {
    float p = a.params[i], m = a.m_par[i], v = a.v_par[i];
    adam_one(p, m, v, g, a.lr_w, a);
    a.params[i] = p;
    a.m_par[i] = m;
    a.v_par[i] = v;
}

__device__ void adam_latent(const AdamParams& a, int64_t j);

__global__ void adam_kernel(const __grid_constant__ AdamParams a) {
    pdl_wait();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < a.P) {  // weights: dense
        adam_weight(a, i, a.grad_par[i]);
        return;
    }
    adam_latent(a, i - a.P);
}

// GRADS|APPLY in one launch after the fused forward/backward: blocks [0, rblocks) reduce the
// weight-gradient partials and apply Adam to the weights they just reduced; the remaining
// blocks apply Adam to the footprint latents (their gradients are complete).
__global__ void __launch_bounds__(256) reduce_adam_kernel(const __grid_constant__ ReduceArgs r,
                                                          const __grid_constant__ AdamParams a, int rblocks) {
    pdl_wait();  // the training kernel's partials and latent gradients are complete
    if ((int)blockIdx.x < rblocks) {
        // the Adam state of this thread's weight is loaded together with the partials (one
        // memory round trip instead of two)
        const int iw = (int)blockIdx.x * 32 + (int)(threadIdx.x & 31);
        const bool own = threadIdx.x < 32 && iw < a.P;
        float pw = 0.0f, mw = 0.0f, vw = 0.0f;
        if (own) {
            pw = a.params[iw];
            mw = a.m_par[iw];
            vw = a.v_par[iw];
        }
        int i;
        const float g = reduce_block(r, blockIdx.x, i);
        if (i >= 0) {
            adam_one(pw, mw, vw, g, a.lr_w, a);
            a.params[i] = pw;
            a.m_par[i] = mw;
            a.v_par[i] = vw;
        }
        return;
    }
    adam_latent(a, (int64_t)(blockIdx.x - rblocks) * blockDim.x + threadIdx.x);
}

__device__ __forceinline__ void adam_latent_one(const AdamParams& a, int64_t li, int bits, bool sparse) {
    const float g = a.grad_lat[li];
    if (sparse && g == 0.0f) return;  // R18: footprint-sparse Adam skips g == 0
    float p = a.latents[li], m = a.m_lat[li], v = a.v_lat[li];
    adam_one(p, m, v, g, a.lr_l, a);
    const float N = (float)(1 << bits);
    p = fminf(fmaxf(p, -(N - 1.0f) / (2.0f * N)), 0.5f);  // clamp to [-(N-1)Q/2, NQ/2]
    a.latents[li] = p;
    a.m_lat[li] = m;
    a.v_lat[li] = v;
}

// latents LPT j .. LPT j + LPT - 1 of the update set (footprint boxes, or every latent)
__device__ void adam_latent(const AdamParams& a, int64_t j) {
    if (a.freeze) return;
    if (a.dense_latents) {
#pragma unroll
        for (int e = 0; e < LPT; ++e) {
            const int64_t li = LPT * j + e;
            if (li >= a.n_latents) return;
            int g = 0;
            while (li >= a.grid_start[g + 1]) ++g;
            adam_latent_one(a, li, a.grid_bits[g], false);
        }
        return;
    }
    const int32_t n = a.box_start[a.nbox];
    const int32_t i = (int32_t)(LPT * j);
    if (i >= n) return;
    int b;
    int64_t li;
    int32_t rem, rw;
    box_locate_row(a.box, a.box_start, a.nbox, i, b, li, rem, rw);
    // addresses and every load first (the stores may alias them as far as the compiler
    // knows), then the updates
    const int ne = min(LPT, n - i);
    int64_t lis[LPT];
    int bits[LPT];
    float g[LPT], pv[LPT], mv[LPT], vv[LPT];
#pragma unroll
    for (int e = 0; e < LPT; ++e) {
        if (e > 0 && e < ne) box_next(a.box, a.box_start, a.nbox, i + e, b, li, rem, rw);
        lis[e] = li;
        bits[e] = a.box[b].bits;
        g[e] = e < ne ? a.grad_lat[li] : 0.0f;
        pv[e] = e < ne ? a.latents[li] : 0.0f;
        mv[e] = e < ne ? a.m_lat[li] : 0.0f;
        vv[e] = e < ne ? a.v_lat[li] : 0.0f;
    }
#pragma unroll
    for (int e = 0; e < LPT; ++e) {
        if (e >= ne || g[e] == 0.0f) continue;  // R18: footprint-sparse Adam skips g == 0
        float pe = pv[e], me = mv[e], ve = vv[e];
        adam_one(pe, me, ve, g[e], a.lr_l, a);
        const float N = (float)(1 << bits[e]);
        pe = fminf(fmaxf(pe, -(N - 1.0f) / (2.0f * N)), 0.5f);  // clamp
        a.latents[lis[e]] = pe;
        a.m_lat[lis[e]] = me;
        a.v_lat[lis[e]] = ve;
    }
}

}  // namespace ntc

// ====================================================================== host side
using namespace ntc;

// launch `kernel` so that it may start while the previous kernel of the stream finishes
// (programmatic dependent launch; the kernel calls pdl_wait() before reading its inputs)
template <class... KArgs, class... Args>
static cudaError_t launch_pdl(void (*kernel)(KArgs...), int grid, int block, uint32_t smem, cudaStream_t st,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

extern "C" int32_t ntc_num_mips(const ntc_desc* d);
extern "C" int32_t ntc_num_levels(const ntc_desc* d);
extern "C" int32_t ntc_level_of_mip(const ntc_desc* d, int32_t mip);
extern "C" int64_t ntc_num_latents(const ntc_desc* d);
extern "C" int64_t ntc_num_params(const ntc_desc* d);
extern "C" ntc_status ntc_grid_layout(const ntc_desc* d, int32_t level, int32_t* r0, int32_t* r1, int64_t* off0,
                                      int64_t* off1);
namespace ntc {
ntc_status api_fail(ntc_status s, const char* msg);
ntc_status check_desc(const ntc_desc* d);
uint16_t host_f16(double v);
double host_tri(double t);
}  // namespace ntc

struct ntc_trainer {
    ntc_desc d;
    int num_sms = 148;
    float* partial = nullptr;
    float* loss_partial = nullptr;
    uint8_t* wimg = nullptr;
};

static int ilog2_t(int64_t v) {
    int l = 0;
    while ((int64_t(1) << (l + 1)) <= v) ++l;
    return l;
}

// compiled training profiles (Table 2) and the kernel instantiation of (profile, act, depth)
static int train_profile(const ntc_desc* d) {
    if (d->c0 == 8 && d->b0 == 2 && d->c1 == 12 && d->b1 == 4) return 0;
    if (d->c0 == 12 && d->b0 == 4 && d->c1 == 20 && d->b1 == 4) return 1;
    if (d->c0 == 12 && d->b0 == 2 && d->c1 == 10 && d->b1 == 4) return 2;
    if (d->c0 == 16 && d->b0 == 4 && d->c1 == 12 && d->b1 == 4) return 3;
    return -1;
}

template <class F>
static void train_dispatch(const ntc_desc* d, F&& f) {
    auto with_ah = [&](auto pr) {
        const bool g = d->activation == 1;
        if (d->hidden_mats == 2)
            g ? f(pr, std::integral_constant<int, 1>{}, std::integral_constant<int, 2>{})
              : f(pr, std::integral_constant<int, 0>{}, std::integral_constant<int, 2>{});
        else
            g ? f(pr, std::integral_constant<int, 1>{}, std::integral_constant<int, 1>{})
              : f(pr, std::integral_constant<int, 0>{}, std::integral_constant<int, 1>{});
    };
    switch (train_profile(d)) {
        case 0: with_ah(Prof<8, 2, 12, 4>{}); break;
        case 1: with_ah(Prof<12, 4, 20, 4>{}); break;
        case 2: with_ah(Prof<12, 2, 10, 4>{}); break;
        default: with_ah(Prof<16, 4, 12, 4>{}); break;
    }
}

extern "C" ntc_status ntc_trainer_create(const ntc_desc* d, ntc_trainer** out) {
    if (!d || !out) return api_fail(NTC_ERR_INVALID_ARGUMENT, "NULL argument");
    if (ntc_status s = check_desc(d)) return s;  // same validation as every decode entry point
    if (train_profile(d) < 0 || (d->hidden_mats != 1 && d->hidden_mats != 2) ||
        (d->activation != 0 && d->activation != 1))
        return api_fail(NTC_ERR_UNSUPPORTED, "training kernel compiled for the Table 2 profiles, depth 1 or 2, hardGELU or GELU");
    if (d->channels < 1 || d->channels > 16 || d->width < 8 || (d->width & (d->width - 1)) ||
        d->width > (1 << 15))
        return api_fail(NTC_ERR_INVALID_ARGUMENT, "bad texture dims");
    auto* t = new ntc_trainer();
    t->d = *d;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&t->num_sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t P = ntc_num_params(d);
    cudaError_t e = cudaMalloc(&t->partial, sizeof(float) * ((P + 3) & ~3) * t->num_sms);
    if (e == cudaSuccess) e = cudaMalloc(&t->loss_partial, sizeof(float) * t->num_sms * TrainSmemT<1>::SLOTS);
    if (e == cudaSuccess) e = cudaMalloc(&t->wimg, TRAIN_WEND_MAX);
    if (e == cudaSuccess) e = cudaMemset(t->wimg, 0, TRAIN_WEND_MAX);
    if (e != cudaSuccess) {
        ntc_trainer_destroy(t);
        return api_fail(NTC_ERR_CUDA, cudaGetErrorString(e));
    }
    *out = t;
    return NTC_OK;
}

extern "C" void ntc_trainer_destroy(ntc_trainer* t) {
    if (!t) return;
    if (t->partial) cudaFree(t->partial);
    if (t->loss_partial) cudaFree(t->loss_partial);
    if (t->wimg) cudaFree(t->wimg);
    delete t;
}

// inclusive tap range [lo, hi] of a grid of resolution r over texels [a, b] of a mip of width 2^lw
static void tap_range(int a, int b, int r, int lw, int* lo, int* hi) {
    const int lr = ilog2_t(r);
    const int na = ((2 * a + 1) << lr) - (1 << lw), nb = ((2 * b + 1) << lr) - (1 << lw);
    *lo = std::max(na >> (lw + 1), 0);
    *hi = std::min((nb >> (lw + 1)) + 1, r - 1);
}

struct Rect {
    int x0, y0, x1, y1;
};

// r minus s as up to four disjoint rectangles
static void rect_subtract(const Rect& r, const Rect& s, std::vector<Rect>& out) {
    if (s.x1 < r.x0 || s.x0 > r.x1 || s.y1 < r.y0 || s.y0 > r.y1) {
        out.push_back(r);
        return;
    }
    if (s.y0 > r.y0) out.push_back({r.x0, r.y0, r.x1, s.y0 - 1});
    if (s.y1 < r.y1) out.push_back({r.x0, s.y1 + 1, r.x1, r.y1});
    const int ya = std::max(r.y0, s.y0), yb = std::min(r.y1, s.y1);
    if (s.x0 > r.x0) out.push_back({r.x0, ya, s.x0 - 1, yb});
    if (s.x1 < r.x1) out.push_back({s.x1 + 1, ya, r.x1, yb});
}

static ntc_status check_batch(const ntc_desc* d, const ntc_batch* b) {
    if (!b || b->n_crops < 1 || b->n_crops > NTC_MAX_CROPS || !b->crops)
        return api_fail(NTC_ERR_INVALID_ARGUMENT, "bad batch (1 <= n_crops <= NTC_MAX_CROPS)");
    if (b->mip < 0 || b->mip >= ntc_num_mips(d)) return api_fail(NTC_ERR_INVALID_ARGUMENT, "batch mip out of range");
    const int wm = d->width >> b->mip;
    for (int k = 0; k < b->n_crops; ++k) {
        const int* c = b->crops + 4 * k;
        if (c[2] < 1 || c[3] < 1 || c[0] < 0 || c[1] < 0 || c[0] + c[2] > wm || c[1] + c[3] > wm)
            return api_fail(NTC_ERR_INVALID_ARGUMENT, "crop outside the mip");
    }
    return NTC_OK;
}

// disjoint footprint boxes of a batch (both grids of the batch's level)
static std::vector<Box> footprint(const ntc_desc* d, const ntc_batch* b) {
    const int j = ntc_level_of_mip(d, b->mip);
    int32_t r[2];
    int64_t off[2];
    ntc_grid_layout(d, j, &r[0], &r[1], &off[0], &off[1]);
    const int lw = ilog2_t(d->width >> b->mip);
    std::vector<Box> boxes;
    for (int k = 0; k < 2; ++k) {
        std::vector<Rect> acc;
        for (int ci = 0; ci < b->n_crops; ++ci) {
            const int* c = b->crops + 4 * ci;
            Rect nr;
            tap_range(c[0], c[0] + c[2] - 1, r[k], lw, &nr.x0, &nr.x1);
            tap_range(c[1], c[1] + c[3] - 1, r[k], lw, &nr.y0, &nr.y1);
            std::vector<Rect> pieces{nr};
            for (const Rect& s : acc) {
                std::vector<Rect> nxt;
                for (const Rect& pc : pieces) rect_subtract(pc, s, nxt);
                pieces.swap(nxt);
            }
            acc.insert(acc.end(), pieces.begin(), pieces.end());
        }
        for (const Rect& q : acc)
            boxes.push_back(Box{off[k], r[k], k ? d->c1 : d->c0, k ? d->b1 : d->b0, q.x0, q.y0, q.x1, q.y1});
    }
    if ((int)boxes.size() > MAX_BOXES) {  // degenerate overlap pattern: one bounding box per grid
        std::vector<Box> bb;
        for (int k = 0; k < 2; ++k) {
            Box u{off[k], r[k], k ? d->c1 : d->c0, k ? d->b1 : d->b0, 1 << 30, 1 << 30, -1, -1};
            for (const Box& x : boxes)
                if (x.off == off[k]) {
                    u.x0 = std::min(u.x0, x.x0);
                    u.y0 = std::min(u.y0, x.y0);
                    u.x1 = std::max(u.x1, x.x1);
                    u.y1 = std::max(u.y1, x.y1);
                }
            bb.push_back(u);
        }
        boxes.swap(bb);
    }
    return boxes;
}

extern "C" int32_t ntc_train_footprint(const ntc_desc* d, const ntc_batch* batch, int32_t* out) {
    if (!d || check_batch(d, batch) != NTC_OK) return -1;
    const std::vector<Box> boxes = footprint(d, batch);
    if (out) {
        const int L = ntc_num_levels(d);
        for (size_t i = 0; i < boxes.size(); ++i) {
            int level = 0, k = 0;
            for (int j = 0; j < L; ++j) {
                int32_t r0, r1;
                int64_t o0, o1;
                ntc_grid_layout(d, j, &r0, &r1, &o0, &o1);
                if (boxes[i].off == o0) level = j, k = 0;
                if (boxes[i].off == o1) level = j, k = 1;
            }
            int32_t* o = out + 6 * i;
            o[0] = level;
            o[1] = k;
            o[2] = boxes[i].x0;
            o[3] = boxes[i].y0;
            o[4] = boxes[i].x1;
            o[5] = boxes[i].y1;
        }
    }
    return (int32_t)boxes.size();
}

// prefix sums of the boxes' latent counts; the kernels index footprints with int32, so a
// footprint past INT32_MAX latents (e.g. one full-mip crop of a 32768^2 NTC 2.25 texture)
// is refused (-1) instead of wrapping
static int32_t box_prefix(const std::vector<Box>& boxes, Box* dst, int32_t* start) {
    int64_t acc = 0;
    for (size_t i = 0; i < boxes.size(); ++i) {
        dst[i] = boxes[i];
        start[i] = (int32_t)acc;
        acc += (int64_t)(boxes[i].x1 - boxes[i].x0 + 1) * (boxes[i].y1 - boxes[i].y0 + 1) * boxes[i].C;
        if (acc > INT32_MAX) return -1;
    }
    start[boxes.size()] = (int32_t)acc;
    return (int32_t)acc;
}
#define FOOTPRINT_TOO_BIG() api_fail(NTC_ERR_UNSUPPORTED, "batch footprint exceeds 2^31-1 latents")

// packed <-> dense copy over footprint boxes (data-parallel latent exchanges):
// mode 0 pack, 1 unpack (src NULL: zero), 2 unpack-add
__global__ void footprint_copy_kernel(const __grid_constant__ PrepParams p, const float* __restrict__ src,
                                      float* __restrict__ dst, int mode) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.box_start[p.nbox]) return;
    int b;
    int64_t li;
    box_locate(p.box, p.box_start, p.nbox, i, b, li);
    if (mode == 1)
        dst[li] = src ? src[i] : 0.0f;
    else if (mode == 2)  // boxes of different senders may overlap: the adds must not race
        atomicAdd(dst + li, src[i]);
    else
        dst[i] = src[li];
}

extern "C" int64_t ntc_footprint_size(const ntc_desc* d, const ntc_batch* batch) {
    if (!d || check_batch(d, batch) != NTC_OK) return -1;
    int64_t n = 0;
    for (const Box& b : footprint(d, batch)) n += (int64_t)(b.x1 - b.x0 + 1) * (b.y1 - b.y0 + 1) * b.C;
    return n;
}

static ntc_status footprint_copy(const ntc_desc* d, const ntc_batch* batch, const float* src, float* dst, int unpack,
                                 ntc_stream stream) {
    if (!d) return api_fail(NTC_ERR_INVALID_ARGUMENT, "NULL desc");
    if (ntc_status s = check_batch(d, batch)) return s;
    if (!dst || (!unpack && !src)) return api_fail(NTC_ERR_INVALID_ARGUMENT, "NULL buffer");
    PrepParams pp;
    memset(&pp, 0, sizeof pp);
    const std::vector<Box> boxes = footprint(d, batch);
    pp.nbox = (int32_t)boxes.size();
    const int32_t n = box_prefix(boxes, pp.box, pp.box_start);
    if (n < 0) return FOOTPRINT_TOO_BIG();
    if (n == 0) return NTC_OK;
    footprint_copy_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(pp, src, dst, unpack);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? NTC_OK : api_fail(NTC_ERR_CUDA, cudaGetErrorString(e));
}

extern "C" ntc_status ntc_footprint_pack(const ntc_desc* d, const ntc_batch* batch, const float* src, float* packed,
                                         ntc_stream stream) {
    return footprint_copy(d, batch, src, packed, 0, stream);
}

extern "C" ntc_status ntc_footprint_unpack(const ntc_desc* d, const ntc_batch* batch, const float* packed,
                                           float* dst, ntc_stream stream) {
    return footprint_copy(d, batch, packed, dst, 1, stream);
}

// ---- explicit box lists (sharded data-parallel mode, DESIGN.md multi-GPU): [n][6] int32
// (level, grid k, x0, y0, x1, y1) inclusive, disjoint
static ntc_status boxes_from_abi(const ntc_desc* d, const int32_t* in, int32_t n, std::vector<Box>& out) {
    if (!d || (n > 0 && !in)) return api_fail(NTC_ERR_INVALID_ARGUMENT, "NULL argument");
    if (n < 0 || n > MAX_BOXES) return api_fail(NTC_ERR_INVALID_ARGUMENT, "box count out of range");
    const int L = ntc_num_levels(d);
    out.clear();
    for (int i = 0; i < n; ++i) {
        const int32_t* b = in + 6 * i;
        if (b[0] < 0 || b[0] >= L || (b[1] != 0 && b[1] != 1)) return api_fail(NTC_ERR_INVALID_ARGUMENT, "bad box grid");
        int32_t r[2];
        int64_t off[2];
        ntc_grid_layout(d, b[0], &r[0], &r[1], &off[0], &off[1]);
        const int k = b[1];
        if (b[2] < 0 || b[3] < 0 || b[2] > b[4] || b[3] > b[5] || b[4] >= r[k] || b[5] >= r[k])
            return api_fail(NTC_ERR_INVALID_ARGUMENT, "box outside its grid");
        out.push_back(Box{off[k], r[k], k ? d->c1 : d->c0, k ? d->b1 : d->b0, b[2], b[3], b[4], b[5]});
    }
    return NTC_OK;
}

extern "C" int64_t ntc_boxes_size(const ntc_desc* d, const int32_t* boxes, int32_t n) {
    std::vector<Box> bx;
    if (boxes_from_abi(d, boxes, n, bx) != NTC_OK) return -1;
    int64_t acc = 0;
    for (const Box& b : bx) acc += (int64_t)(b.x1 - b.x0 + 1) * (b.y1 - b.y0 + 1) * b.C;
    return acc;
}

extern "C" ntc_status ntc_boxes_copy(const ntc_desc* d, const int32_t* boxes, int32_t n, const float* src,
                                     float* dst, int32_t mode, ntc_stream stream) {
    std::vector<Box> bx;
    if (ntc_status s = boxes_from_abi(d, boxes, n, bx)) return s;
    if (mode < NTC_BOX_PACK || mode > NTC_BOX_ZERO) return api_fail(NTC_ERR_INVALID_ARGUMENT, "bad mode");
    if (!dst || (mode != NTC_BOX_ZERO && !src)) return api_fail(NTC_ERR_INVALID_ARGUMENT, "NULL buffer");
    PrepParams pp;
    memset(&pp, 0, sizeof pp);
    pp.nbox = (int32_t)bx.size();
    const int32_t cnt = box_prefix(bx, pp.box, pp.box_start);
    if (cnt < 0) return FOOTPRINT_TOO_BIG();
    if (cnt == 0) return NTC_OK;
    const int km = mode == NTC_BOX_PACK ? 0 : mode == NTC_BOX_ADD ? 2 : 1;
    footprint_copy_kernel<<<(cnt + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
        pp, mode == NTC_BOX_ZERO ? nullptr : src, dst, km);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? NTC_OK : api_fail(NTC_ERR_CUDA, cudaGetErrorString(e));
}

static ntc_status apply_step(const ntc_desc* d, const ntc_train_buffers* buf, const std::vector<Box>& boxes,
                             const ntc_train_hparams* hp, cudaStream_t st);
static int64_t build_adam(const ntc_desc* d, const ntc_train_buffers* buf, const std::vector<Box>& boxes,
                          const ntc_train_hparams* hp, AdamParams& a);
static bool apply_buffers_ok(const ntc_train_buffers* buf);

extern "C" ntc_status ntc_train_apply_boxes(ntc_trainer* t, const ntc_desc* d, const ntc_train_buffers* buf,
                                            const int32_t* boxes, int32_t n, const ntc_train_hparams* hp,
                                            ntc_stream stream) {
    if (!t || !d || !buf || !hp) return api_fail(NTC_ERR_INVALID_ARGUMENT, "NULL argument");
    if (memcmp(&t->d, d, sizeof(ntc_desc)) != 0) return api_fail(NTC_ERR_INVALID_ARGUMENT, "desc != trainer desc");
    if (hp->step < 1) return api_fail(NTC_ERR_INVALID_ARGUMENT, "step must be >= 1");
    std::vector<Box> bx;
    if (ntc_status s = boxes_from_abi(d, boxes, n, bx)) return s;
    return apply_step(d, buf, bx, hp, (cudaStream_t)stream);
}

extern "C" ntc_status ntc_train_step(ntc_trainer* t, const ntc_desc* d, const ntc_train_buffers* buf,
                                     const ntc_batch* batch, const ntc_train_hparams* hp, float* loss,
                                     int32_t* status, uint32_t flags, ntc_stream stream) {
    if (!t || !d || !buf || !hp) return api_fail(NTC_ERR_INVALID_ARGUMENT, "NULL argument");
    if (memcmp(&t->d, d, sizeof(ntc_desc)) != 0) return api_fail(NTC_ERR_INVALID_ARGUMENT, "desc != trainer desc");
    if (ntc_status s = check_batch(d, batch)) return s;
    if (hp->step < 1) return api_fail(NTC_ERR_INVALID_ARGUMENT, "step must be >= 1");
    cudaStream_t st = (cudaStream_t)stream;
    const std::vector<Box> boxes = footprint(d, batch);
    const int64_t P = ntc_num_params(d), NL = ntc_num_latents(d);
    cudaError_t e = cudaSuccess;
    if (flags & NTC_STEP_GRADS) {
        if (!buf->latents || !buf->noisy || !buf->grad_lat || !buf->params || !buf->grad_par || !loss || !batch->ref)
            return api_fail(NTC_ERR_INVALID_ARGUMENT, "NULL buffer");
        if (reinterpret_cast<uintptr_t>(batch->ref) & 3)  // read as aligned 32-bit words
            return api_fail(NTC_ERR_INVALID_ARGUMENT, "reference image must be 4-byte aligned");
        // t2: noisy latents + zeroed gradients over the footprint
        PrepParams pp;
        memset(&pp, 0, sizeof pp);
        pp.nbox = (int32_t)boxes.size();
        const int32_t n = box_prefix(boxes, pp.box, pp.box_start);
        if (n < 0) return FOOTPRINT_TOO_BIG();
        pp.latents = buf->latents;
        pp.noisy = reinterpret_cast<__half*>(buf->noisy);
        pp.grad_lat = buf->grad_lat;
        pp.seed = hp->seed;
        pp.step = (uint32_t)hp->step;
        pp.noise_on = hp->noise_on;
        if (hp->dense_latent_adam) cudaMemsetAsync(buf->grad_lat, 0, sizeof(float) * NL, st);
        pp.prep_blocks = (int32_t)((n + 256 * LPT - 1) / (256 * LPT));
        pp.params = buf->params;
        pp.D = 4 * d->c0 + d->c1 + 13;
        pp.c = d->channels;
        pp.hm = d->hidden_mats;
        pp.wimg = t->wimg;
        {
            const int pg = pp.prep_blocks + (wimg_items(pp.hm, pp.D + 1 > 64 ? 2 : 1) + 255) / 256;
            if (TRAIN_PREP_PDL) {  // overlaps this launch with the previous kernel's tail
                const cudaError_t e = launch_pdl(prep_kernel, pg, 256, 0, st, pp);
                if (e != cudaSuccess) return api_fail(NTC_ERR_CUDA, cudaGetErrorString(e));
            } else {
                prep_kernel<<<pg, 256, 0, st>>>(pp);
            }
        }
        // t1, t3-t7
        TrainParams tp;
        memset(&tp, 0, sizeof tp);
        const int m = batch->mip;
        const int j = ntc_level_of_mip(d, m);
        int32_t r0, r1;
        int64_t o0, o1;
        ntc_grid_layout(d, j, &r0, &r1, &o0, &o1);
        tp.W = d->width;
        tp.c = d->channels;
        tp.M = ntc_num_mips(d);
        tp.mip = m;
        tp.lw = tp.M - 1 - m;
        tp.r0 = r0;
        tp.r1 = r1;
        tp.lr0 = ilog2_t(r0);
        tp.lr1 = ilog2_t(r1);
        tp.off0 = o0;
        tp.off1 = o1;
        const double lod = tp.M > 1 ? (double)m / (double)(tp.M - 1) : 0.0;  // R6
        tp.lod_word = (uint32_t)host_f16(lod) | ((uint32_t)host_f16(1.0) << 16);
        for (int qq = 0; qq < 8; ++qq) {
            uint16_t v[6];
            for (int h = 0; h < 3; ++h) {
                const double tt = (double)(1 << h) * qq / 8.0;
                v[2 * h] = host_f16(host_tri(tt));
                v[2 * h + 1] = host_f16(host_tri(tt - 0.25));
            }
            for (int k = 0; k < 3; ++k) tp.pe_words[qq][k] = (uint32_t)v[2 * k] | ((uint32_t)v[2 * k + 1] << 16);
        }
        tp.n_crops = batch->n_crops;
        int64_t B = 0, tiles = 0;
        for (int k = 0; k < batch->n_crops; ++k) {
            for (int f = 0; f < 4; ++f) tp.crop[k][f] = batch->crops[4 * k + f];
            tp.tile_start[k] = (int32_t)tiles;
            const int64_t area = (int64_t)batch->crops[4 * k + 2] * batch->crops[4 * k + 3];
            B += area;
            tiles += (area + TILE_M - 1) / TILE_M;
        }
        for (int k = batch->n_crops; k <= NTC_MAX_CROPS; ++k) tp.tile_start[k] = INT32_MAX;
        tp.tile_start[batch->n_crops] = (int32_t)tiles;
        tp.n_tiles = (int32_t)tiles;
        tp.ref = batch->ref;
        tp.ref_stride = batch->ref_row_stride_elems;
        const int64_t Bn = batch->norm_texels > 0 ? batch->norm_texels : B;
        tp.inv_bc = (float)(1.0 / ((double)Bn * d->channels));
        tp.noisy = reinterpret_cast<const __half*>(buf->noisy);
        tp.grad_lat = buf->grad_lat;
        tp.wimg = t->wimg;
        tp.partial = t->partial;
        tp.loss_partial = t->loss_partial;
        tp.P = (int32_t)P;
        tp.Pst = (int32_t)((P + 3) & ~3);
        tp.freeze = hp->freeze_latents;
        int slots = 1;
        uint32_t smem_bytes = 0;
        void (*k)(TrainParams) = nullptr;
        train_dispatch(d, [&](auto pr, auto a, auto h) {
            using PP = decltype(pr);
            constexpr int A = decltype(a)::value, H = decltype(h)::value;
            using SS = TrainSmemT<H, TrainGeom<PP>::KA>;
            slots = SS::SLOTS;
            smem_bytes = SS::BYTES;
            k = train_kernel<PP, A, H>;
            // the bench's training material (NTC 0.2, [57,64,64,9], hardGELU): channel count
            // compiled in
            if constexpr (std::is_same<PP, Prof<8, 2, 12, 4>>::value && A == 0 && H == 1)
                if (d->channels == 9) k = train_kernel<PP, 0, 1, 9>;
        });
        const int grid = (int)std::min<int64_t>(std::min<int64_t>(t->num_sms, 8 * RED_MAXK),
                                                (tiles + slots - 1) / slots);
        e = ensure_smem((const void*)k, smem_bytes);
        if (e == cudaSuccess) {
            e = launch_pdl(k, grid, slots * 256, smem_bytes, st, tp);
            if (e != cudaSuccess) return api_fail(NTC_ERR_CUDA, cudaGetErrorString(e));
            // t6: deterministic cross-CTA reduction, scaled by 1/(B c); with APPLY in the same
            // call, t8 rides in the same launch (weights Adam'd as they are reduced)
            const ReduceArgs ra{t->partial,  (size_t)tp.Pst,  t->loss_partial, grid, (int)P, grid * slots,
                                tp.inv_bc,   buf->grad_par, loss,         status};
            const int rblocks = (int)((P + 31) / 32);
            if ((flags & NTC_STEP_APPLY) && apply_buffers_ok(buf)) {
                AdamParams a;
                const int64_t nlat = build_adam(d, buf, boxes, hp, a);
                if (nlat < 0) return FOOTPRINT_TOO_BIG();
                e = launch_pdl(reduce_adam_kernel, rblocks + (int)((nlat + 256 * LPT - 1) / (256 * LPT)), 256, 0, st,
                               ra, a, rblocks);
                if (e != cudaSuccess) return api_fail(NTC_ERR_CUDA, cudaGetErrorString(e));
                return NTC_OK;
            }
            e = launch_pdl(reduce_kernel, rblocks, 256, 0, st, ra);
        }
        if (e != cudaSuccess) return api_fail(NTC_ERR_CUDA, cudaGetErrorString(e));
    }
    if (flags & NTC_STEP_APPLY) return apply_step(d, buf, boxes, hp, st);
    return NTC_OK;
}

// t8 parameters: Adam on the weights (dense) and on the latents of `boxes` (footprint-sparse
// unless dense_latent_adam), then the latent clamp.  Returns the latent work-item count.
static int64_t build_adam(const ntc_desc* d, const ntc_train_buffers* buf, const std::vector<Box>& boxes,
                          const ntc_train_hparams* hp, AdamParams& a) {
    const int64_t P = ntc_num_params(d), NL = ntc_num_latents(d);
    memset(&a, 0, sizeof a);
    a.nbox = (int32_t)boxes.size();
    const int32_t n = box_prefix(boxes, a.box, a.box_start);
    if (n < 0) return -1;
    a.dense_latents = hp->dense_latent_adam;
    a.n_latents = NL;
    a.P = (int32_t)P;
    a.params = buf->params;
    a.m_par = buf->m_par;
    a.v_par = buf->v_par;
    a.grad_par = buf->grad_par;
    a.latents = buf->latents;
    a.m_lat = buf->m_lat;
    a.v_lat = buf->v_lat;
    a.grad_lat = buf->grad_lat;
    a.lr_w = hp->lr_weight;
    a.lr_l = hp->lr_latent;
    a.freeze = hp->freeze_latents;
    a.b1 = hp->beta1;
    a.b2 = hp->beta2;
    a.eps = hp->eps;
    a.c1 = (float)(1.0 - std::pow((double)hp->beta1, (double)hp->step));
    a.c2 = (float)(1.0 - std::pow((double)hp->beta2, (double)hp->step));
    const int L = ntc_num_levels(d);
    a.ngrid = 2 * L;
    int64_t acc = 0;
    for (int j = 0; j < L; ++j) {
        int32_t r0, r1;
        int64_t o0, o1;
        ntc_grid_layout(d, j, &r0, &r1, &o0, &o1);
        a.grid_start[2 * j] = o0;
        a.grid_bits[2 * j] = d->b0;
        a.grid_start[2 * j + 1] = o1;
        a.grid_bits[2 * j + 1] = d->b1;
        acc = o1 + (int64_t)r1 * r1 * d->c1;
    }
    a.grid_start[2 * L] = acc;
    return hp->freeze_latents ? 0 : (hp->dense_latent_adam ? NL : (int64_t)n);
}

static bool apply_buffers_ok(const ntc_train_buffers* buf) {
    return buf->latents && buf->m_lat && buf->v_lat && buf->grad_lat && buf->params && buf->m_par && buf->v_par &&
           buf->grad_par;
}

static ntc_status apply_step(const ntc_desc* d, const ntc_train_buffers* buf, const std::vector<Box>& boxes,
                             const ntc_train_hparams* hp, cudaStream_t st) {
    if (!apply_buffers_ok(buf)) return api_fail(NTC_ERR_INVALID_ARGUMENT, "NULL buffer");
    AdamParams a;
    const int64_t nlat = build_adam(d, buf, boxes, hp, a);
    if (nlat < 0) return FOOTPRINT_TOO_BIG();
    const int64_t total = ntc_num_params(d) + (nlat + LPT - 1) / LPT;
    adam_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(a);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? NTC_OK : api_fail(NTC_ERR_CUDA, cudaGetErrorString(e));
}
