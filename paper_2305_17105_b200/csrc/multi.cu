// multi.cu -- multi-material random-access decode, product code.
//
// The paper handles neighbouring pixels of different materials inside one shader wave with a
// wave-intrinsic loop over the distinct materials.  On B200 the unit of
// execution is a 128-texel tcgen05 tile that multiplies ONE weight set, so the queries are
// bucketed by material first:
//   count    per-material histogram (SMEM per block, one global add per bin and block);
//            queries with a material index >= n_mats get their NaN row and the status bit
//   scan     one block: query offsets `seg` and 128-texel tile offsets `tstart` per material
//   scatter  each block reserves a contiguous slot range per material with one global add
//            and writes the query indices there (perm)
//   decode   decode_multi_kernel: each persistent CTA takes a contiguous share of the
//            material-sorted tile list and swaps the SMEM weight image at material edges.
// Outputs go to each query's own row, so the (unordered) slot order inside a material does
// not affect any result.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "material.h"

namespace ntc {
ntc_status api_fail(ntc_status s, const char* msg);
DecodeParams base_params(const ntc_material* m);
cudaError_t launch_decode_multi(int pid, int hm, const DecodeParams& p, const MultiTable& mt, int grid,
                                cudaStream_t s);

namespace {
// scratch layout (bytes)
constexpr int64_t OFF_COUNT = 0, OFF_SEG = 1024, OFF_TSTART = 2112, OFF_CURSOR = 3200, OFF_PERM = 4352;
constexpr int MULTI_ITEMS = 8;  // queries per thread in the scatter pass

// SMEM counter add with a warp fast path: when every active lane has the same key (long runs
// in screen-ordered query streams) one atomic serves the warp; otherwise one atomic per lane.
// Returns this lane's slot (old value + rank among the lanes sharing the key).
__device__ __forceinline__ int agg_add(int32_t* h, int key, bool active) {
    const unsigned act = __ballot_sync(0xFFFFFFFFu, active);
    if (act == 0) return 0;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(act) - 1;
    const int k0 = __shfl_sync(0xFFFFFFFFu, key, leader);
    if (__all_sync(0xFFFFFFFFu, !active || key == k0)) {
        int base = 0;
        if (lane == leader) base = atomicAdd(&h[k0], __popc(act));
        base = __shfl_sync(0xFFFFFFFFu, base, leader);
        return base + __popc(act & ((1u << lane) - 1u));
    }
    return active ? atomicAdd(&h[key], 1) : 0;
}

__global__ void multi_count_kernel(const ntc_query* __restrict__ q, int64_t n, int n_mats, int c,
                                   int32_t* __restrict__ count, uint16_t* __restrict__ out,
                                   int32_t* __restrict__ status) {
    __shared__ int32_t h[NTC_MAX_MATERIALS];
    for (int i = threadIdx.x; i < NTC_MAX_MATERIALS; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * blockDim.x * MULTI_ITEMS;
    int mat[MULTI_ITEMS];
#pragma unroll
    for (int k = 0; k < MULTI_ITEMS; ++k) {  // all loads in flight first
        const int64_t i = base + (int64_t)k * blockDim.x + threadIdx.x;
        mat[k] = i < n ? (int)((__ldg(reinterpret_cast<const uint2*>(q) + i).y >> 8) & 0xFFu) : -1;
    }
    bool badseen = false;
#pragma unroll
    for (int k = 0; k < MULTI_ITEMS; ++k) {
        const int64_t i = base + (int64_t)k * blockDim.x + threadIdx.x;
        agg_add(h, mat[k] >= 0 && mat[k] < n_mats ? mat[k] : 0, mat[k] >= 0 && mat[k] < n_mats);
        if (mat[k] >= n_mats) {
            for (int j = 0; j < c; ++j) out[i * c + j] = 0x7E00u;  // NaN row
            badseen = true;
        }
    }
    if (badseen && status) atomicOr(status, (int)NTC_ERR_OUT_OF_RANGE);
    __syncthreads();
    for (int i = threadIdx.x; i < n_mats; i += blockDim.x)
        if (h[i]) atomicAdd(&count[i], h[i]);
}

// exclusive scans of the counts and of their 128-texel tile counts (n_mats <= 256 = blockDim)
__global__ void multi_scan_kernel(const int32_t* __restrict__ count, int n_mats, int32_t* __restrict__ seg,
                                  int32_t* __restrict__ tstart, int32_t* __restrict__ cursor) {
    __shared__ int32_t sc[NTC_MAX_MATERIALS], st[NTC_MAX_MATERIALS];
    const int t = threadIdx.x;
    const int32_t cnt = t < n_mats ? count[t] : 0;
    sc[t] = cnt;
    st[t] = (cnt + TILE_M - 1) / TILE_M;
    __syncthreads();
    for (int d = 1; d < NTC_MAX_MATERIALS; d <<= 1) {  // Hillis-Steele inclusive scan
        const int32_t a = t >= d ? sc[t - d] : 0, b = t >= d ? st[t - d] : 0;
        __syncthreads();
        sc[t] += a;
        st[t] += b;
        __syncthreads();
    }
    if (t < n_mats) {
        seg[t + 1] = sc[t];
        tstart[t + 1] = st[t];
        cursor[t] = sc[t] - cnt;
    }
    if (t == 0) {
        seg[0] = 0;
        tstart[0] = 0;
    }
}

__global__ void multi_scatter_kernel(const ntc_query* __restrict__ q, int64_t n, int n_mats,
                                     int32_t* __restrict__ cursor, int32_t* __restrict__ perm) {
    __shared__ int32_t h[NTC_MAX_MATERIALS];
    for (int i = threadIdx.x; i < NTC_MAX_MATERIALS; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * blockDim.x * MULTI_ITEMS;
    int mat[MULTI_ITEMS], rank[MULTI_ITEMS];
#pragma unroll
    for (int k = 0; k < MULTI_ITEMS; ++k) {
        const int64_t i = base + (int64_t)k * blockDim.x + threadIdx.x;
        const int m = i < n ? (int)((__ldg(reinterpret_cast<const uint2*>(q) + i).y >> 8) & 0xFFu) : n_mats;
        const bool ok = m < n_mats;
        mat[k] = ok ? m : -1;
        rank[k] = agg_add(h, ok ? m : 0, ok);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n_mats; i += blockDim.x)
        if (h[i]) h[i] = atomicAdd(&cursor[i], h[i]);  // block's first slot of material i
    __syncthreads();
#pragma unroll
    for (int k = 0; k < MULTI_ITEMS; ++k)
        if (mat[k] >= 0) perm[h[mat[k]] + rank[k]] = (int32_t)(base + (int64_t)k * blockDim.x + threadIdx.x);
}
}  // namespace
}  // namespace ntc

using namespace ntc;

extern "C" int64_t ntc_decode_multi_scratch_bytes(int64_t n) { return OFF_PERM + 4 * (n > 0 ? n : 0); }

extern "C" ntc_status ntc_decode_texels_multi(const ntc_material* const* mats, int32_t n_mats, const ntc_query* q,
                                              int64_t n, uint16_t* out, int32_t* status, void* scratch,
                                              int64_t scratch_bytes, ntc_stream stream) {
    if (!mats || n_mats < 1 || n_mats > NTC_MAX_MATERIALS)
        return api_fail(NTC_ERR_INVALID_ARGUMENT, "n_mats must be in [1, NTC_MAX_MATERIALS]");
    for (int i = 0; i < n_mats; ++i) {
        if (!mats[i]) return api_fail(NTC_ERR_INVALID_ARGUMENT, "NULL material");
        if (memcmp(&mats[i]->d, &mats[0]->d, sizeof(ntc_desc)) != 0)
            return api_fail(NTC_ERR_INVALID_ARGUMENT, "materials of one multi decode must share one ntc_desc");
    }
    if (n < 0 || n > 0x7FFFFFFF) return api_fail(NTC_ERR_INVALID_ARGUMENT, "n out of range");
    if (n == 0) return NTC_OK;
    if (!q || !out || !scratch) return api_fail(NTC_ERR_INVALID_ARGUMENT, "NULL buffer");
    if (scratch_bytes < ntc_decode_multi_scratch_bytes(n) || (reinterpret_cast<uintptr_t>(scratch) & 15))
        return api_fail(NTC_ERR_INVALID_ARGUMENT, "scratch too small or misaligned");
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t* sb = static_cast<uint8_t*>(scratch);
    int32_t* count = reinterpret_cast<int32_t*>(sb + OFF_COUNT);
    int32_t* seg = reinterpret_cast<int32_t*>(sb + OFF_SEG);
    int32_t* tstart = reinterpret_cast<int32_t*>(sb + OFF_TSTART);
    int32_t* cursor = reinterpret_cast<int32_t*>(sb + OFF_CURSOR);
    int32_t* perm = reinterpret_cast<int32_t*>(sb + OFF_PERM);
    const ntc_material* m0 = mats[0];
    cudaError_t e = cudaMemsetAsync(count, 0, 4 * NTC_MAX_MATERIALS, st);
    if (e != cudaSuccess) return api_fail(NTC_ERR_CUDA, cudaGetErrorString(e));
    const int64_t per = 256 * MULTI_ITEMS;
    multi_count_kernel<<<(int)((n + per - 1) / per), 256, 0, st>>>(q, n, n_mats, m0->d.channels, count, out,
                                                                    status);
    multi_scan_kernel<<<1, NTC_MAX_MATERIALS, 0, st>>>(count, n_mats, seg, tstart, cursor);
    multi_scatter_kernel<<<(int)((n + per - 1) / per), 256, 0, st>>>(q, n, n_mats, cursor, perm);
    e = cudaGetLastError();
    if (e != cudaSuccess) return api_fail(NTC_ERR_CUDA, cudaGetErrorString(e));

    DecodeParams p = base_params(m0);
    p.mode = 1;
    p.q = q;
    p.nq = n;
    p.out = out;
    p.status = status;
    static thread_local MultiTable mt;  // ~20 KB: off the stack; the launch copies it
    memset(&mt, 0, sizeof mt);
    mt.n_mats = n_mats;
    mt.seg = seg;
    mt.tstart = tstart;
    mt.perm = perm;
    for (int i = 0; i < n_mats; ++i) {
        mt.rec[i].grids = mats[i]->grids;
        mt.rec[i].wimg = mats[i]->wimg;
        memcpy(mt.rec[i].b3, mats[i]->b3, sizeof mt.rec[i].b3);
    }
    // total tiles <= n/128 + n_mats; at most one CTA per SM, >= 8 tiles per CTA
    const int64_t tiles_max = (n + TILE_M - 1) / TILE_M + n_mats;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(m0->num_sms, (tiles_max + 7) / 8));
    e = launch_decode_multi(m0->pid, m0->d.hidden_mats, p, mt, grid, st);
    return e == cudaSuccess ? NTC_OK : api_fail(NTC_ERR_CUDA, cudaGetErrorString(e));
}
