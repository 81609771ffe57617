// common.cuh -- shared host/device definitions of the NTC CUDA path (product code).
#pragma once
#include <cstdint>
#include <mutex>
#include <set>
#include <utility>

#include <cuda_runtime.h>

#include "../../include/ntc.h"

namespace ntc {

constexpr int HID = 64;          // hidden width
constexpr int MAX_MIPS = 16;     // W <= 2^15
constexpr int MAX_LEVELS = 8;
constexpr int TILE_M = 128;      // texels per tcgen05 tile (MMA M)
constexpr int NWG = 4;           // warpgroups per decode CTA, each owns a tile pipeline

__host__ __device__ constexpr int pow2_bytes(int bits) {
    return bits <= 8 ? 1 : bits <= 16 ? 2 : bits <= 32 ? 4 : bits <= 64 ? 8 : 16;
}

// Compile-time profile (Table 2): C0 x B0 and C1 x B1 latents, input width D.
template <int C0_, int B0_, int C1_, int B1_>
struct Prof {
    static constexpr int C0 = C0_, B0 = B0_, C1 = C1_, B1 = B1_;
    static constexpr int D = 4 * C0 + C1 + 12 + 1;
    static constexpr int K1 = ((D + 1 + 15) / 16) * 16;  // + the constant-1 bias column
    static constexpr int K1W = K1 / 2;                   // fp16 pairs
    static constexpr int K1_ATOMS = (K1 + 63) / 64;      // 64-wide SW128 atoms along K
    static constexpr int CELL0 = pow2_bytes(C0 * B0);    // packed cell bytes
    static constexpr int CELL1 = pow2_bytes(C1 * B1);
    static_assert((C0 % 2) == 0 && (C1 % 2) == 0, "even channel counts");
    static_assert(32 % B0 == 0 && 32 % B1 == 0, "bits must divide 32");
};

// Per-level geometry for the device: resolutions and byte offsets into the packed grids.
struct LevelGeom {
    int32_t r0, r1;
    int32_t lr0, lr1;    // log2 of r0, r1
    int64_t off0, off1;  // byte offsets of packed G0 / G1 of this level
};

// Everything a decode launch needs, passed by value (param space / constant bank).
struct DecodeParams {
    const uint8_t* grids;
    const uint4* wimg;        // global copy of the SMEM weight image
    uint32_t wimg_bytes;
    int32_t W, c, M, L;
    int32_t mode;             // 0: tiles over mips, 1: queries, 2: debug assemble
    int32_t act;              // 0: hardGELU, 1: exact GELU (selects the kernel instantiation)
    LevelGeom lv[MAX_LEVELS];
    int8_t level_of[MAX_MIPS];
    uint32_t lod_word[MAX_MIPS];  // half(lod) | half(1.0) << 16
    uint32_t pe_words[8][4];      // PE of one axis at p = x mod 8, as 3 half2 words (+pad)
    // mode 0
    int32_t mip_first, mip_count;
    int32_t tile_start[MAX_MIPS + 1];
    int64_t out_off[MAX_MIPS];     // element offset of mip in out
    int64_t row_stride[MAX_MIPS];  // elements
    int32_t n_tiles;     // end of the tile range (exclusive)
    int32_t tile_first;  // start of the tile range (multi-GPU part)
    // mode 1 / 2
    const ntc_query* q;
    int64_t nq;
    int32_t* status;
    int32_t* dbg_addr;
    uint16_t* dbg_X;
    uint16_t* out;
    // paired odd-c stores (decode.cu store_output) for tiles < pair_tiles: those tiles' rows
    // are consecutive output rows starting 4-byte aligned (mode 0: the mips of width >= 128
    // with even offsets and strides, which come first; mode 1: the full tiles)
    int32_t pair_tiles;
    // mode 0: tiles < lin_tiles write output row (tile * 128 + row) of `out` (whole-tile mips
    // laid out back to back from out_off 0, rows of w_m * c elements)
    int32_t lin_tiles;
    // mode 0: tiles < tma_tiles (whole-tile mips, 16-byte aligned `out`) are staged in SMEM and
    // written by one bulk TMA store per tile (decode.cu, DECODE_TMA_OUT)
    int32_t tma_tiles;
    float b3[16];                  // output bias, added in the output epilogue
};

// Multi-material decode: per-material device records in the parameter
// space; the bucketing of the queries by material lives in device scratch (multi.cu).
struct MatRec {
    const uint8_t* grids;
    const uint4* wimg;
    float b3[16];
};
struct MultiTable {
    int32_t n_mats;
    const int32_t* seg;     // [n_mats + 1] offsets of each material's queries in perm
    const int32_t* tstart;  // [n_mats + 1] first tile of each material; [n_mats] = total tiles
    const int32_t* perm;    // query indices grouped by material
    MatRec rec[NTC_MAX_MATERIALS];
};

// Raise a kernel's dynamic-SMEM limit once per (device, kernel, size) instead of on every
// launch (cudaFuncSetAttribute is a driver call; the hot-path entry points are called per step).
inline cudaError_t ensure_smem(const void* kernel, uint32_t bytes) {
    static std::mutex mu;
    static std::set<std::pair<std::pair<int, const void*>, uint32_t>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_pair(std::make_pair(dev, kernel), bytes);
    std::lock_guard<std::mutex> g(mu);
    if (done.count(key)) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done.insert(key);
    return e;
}

}  // namespace ntc
