// api.cu -- the C ABI (include/ntc.h): host-side validation, geometry, material upload,
// decode launches.  Product code; no dependency on the oracle.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "ptx.cuh"

namespace ntc {
int profile_id(const ntc_desc* d);
uint32_t decode_wimg_bytes(int pid, int hm);
cudaError_t build_wimg(int pid, int hm, const uint16_t* w, int c, uint8_t* img, cudaStream_t s);
cudaError_t launch_decode(int pid, int hm, const DecodeParams& p, int grid, cudaStream_t s);
cudaError_t launch_debug_assemble(int pid, const DecodeParams& p, cudaStream_t s);
}  // namespace ntc

using namespace ntc;

static thread_local std::string g_err;

static ntc_status fail(ntc_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

static ntc_status cuda_fail(cudaError_t e, const char* what) {
    return fail(NTC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

extern "C" const char* ntc_last_error(void) { return g_err.c_str(); }

namespace ntc {
ntc_status api_fail(ntc_status s, const char* msg) { return fail(s, "%s", msg); }
}  // namespace ntc

// ------------------------------------------------------------------ geometry
static int ilog2i(int64_t v) {
    int l = 0;
    while ((int64_t(1) << (l + 1)) <= v) ++l;
    return l;
}

namespace ntc {
ntc_status check_desc(const ntc_desc* d) {
    if (!d) return fail(NTC_ERR_INVALID_ARGUMENT, "desc is NULL");
    if (d->width < 4 || d->width > (1 << 15) || (d->width & (d->width - 1)))
        return fail(NTC_ERR_INVALID_ARGUMENT, "width %d must be a power of two in [4, 32768]", d->width);
    if (d->channels < 1 || d->channels > 16) return fail(NTC_ERR_INVALID_ARGUMENT, "channels %d not in [1,16]", d->channels);
    if (d->g0_ratio != 2 && d->g0_ratio != 4) return fail(NTC_ERR_INVALID_ARGUMENT, "g0_ratio must be 2 or 4");
    if (d->width / d->g0_ratio < 2) return fail(NTC_ERR_INVALID_ARGUMENT, "width too small for the profile");
    if (d->b0 < 1 || d->b0 > 8 || d->b1 < 1 || d->b1 > 8 || d->c0 < 1 || d->c1 < 1)
        return fail(NTC_ERR_INVALID_ARGUMENT, "bad grid channels/bits");
    if (d->hidden_mats != 1 && d->hidden_mats != 2) return fail(NTC_ERR_INVALID_ARGUMENT, "hidden_mats must be 1 or 2");
    if (d->activation != 0 && d->activation != 1)
        return fail(NTC_ERR_UNSUPPORTED, "activation must be 0 (hardGELU) or 1 (exact GELU)");
    if (profile_id(d) < 0) return fail(NTC_ERR_UNSUPPORTED, "profile (C0=%d,B0=%d,C1=%d,B1=%d) not compiled", d->c0, d->b0, d->c1, d->b1);
    return NTC_OK;
}
}  // namespace ntc

extern "C" int32_t ntc_num_mips(const ntc_desc* d) { return ilog2i(d->width) + 1; }

extern "C" int32_t ntc_num_levels(const ntc_desc* d) {
    int32_t L = 0;
    for (int64_t r = d->width / d->g0_ratio; r >= 2; r /= 4) ++L;  // G1 = r/2 >= 1 (R7)
    // ... and no level past the one holding the bottom 2-3 mips (R7)
    const int32_t Lm = (ilog2i(d->width) - 1) / 2 > 1 ? (ilog2i(d->width) - 1) / 2 : 1;  // ceil((M-3)/2)
    return L < Lm ? L : Lm;
}

extern "C" int32_t ntc_level_of_mip(const ntc_desc* d, int32_t mip) {
    const int32_t last = ntc_num_levels(d) - 1;
    const int32_t j = mip <= 3 ? 0 : (mip - 2) / 2;  // 0-3 | pairs | tail
    return j < last ? j : last;
}

static void level_res(const ntc_desc* d, int j, int32_t* r0, int32_t* r1) {
    int64_t r = d->width / d->g0_ratio;
    r >>= 2 * j;
    *r0 = (int32_t)r;
    *r1 = (int32_t)(r >= 4 ? r / 2 : 1);
}

extern "C" ntc_status ntc_grid_layout(const ntc_desc* d, int32_t level, int32_t* r0, int32_t* r1, int64_t* off0,
                                      int64_t* off1) {
    if (!d || level < 0 || level >= ntc_num_levels(d)) return fail(NTC_ERR_INVALID_ARGUMENT, "bad level");
    int64_t off = 0;
    for (int j = 0; j <= level; ++j) {
        int32_t a, b;
        level_res(d, j, &a, &b);
        if (j == level) {
            if (r0) *r0 = a;
            if (r1) *r1 = b;
            if (off0) *off0 = off;
            if (off1) *off1 = off + (int64_t)a * a * d->c0;
        }
        off += (int64_t)a * a * d->c0 + (int64_t)b * b * d->c1;
    }
    return NTC_OK;
}

extern "C" int64_t ntc_num_latents(const ntc_desc* d) {
    int64_t n = 0;
    for (int j = 0; j < ntc_num_levels(d); ++j) {
        int32_t a, b;
        level_res(d, j, &a, &b);
        n += (int64_t)a * a * d->c0 + (int64_t)b * b * d->c1;
    }
    return n;
}

extern "C" int64_t ntc_num_params(const ntc_desc* d) {
    const int64_t D = 4 * d->c0 + d->c1 + 13;
    return D * HID + HID + (int64_t)d->hidden_mats * (HID * HID + HID) + (int64_t)HID * d->channels + d->channels;
}

extern "C" int64_t ntc_mip_offset(const ntc_desc* d, int32_t mip) {
    int64_t off = 0;
    for (int m = 0; m < mip; ++m) {
        const int64_t w = d->width >> m;
        off += w * w;
    }
    return off;
}

extern "C" int64_t ntc_chain_texels(const ntc_desc* d) { return ntc_mip_offset(d, ntc_num_mips(d)); }

// ------------------------------------------------------------------ a0: quantise (bit-exact)
struct GridTable {
    int32_t n;
    int64_t start[2 * MAX_LEVELS + 1];
    int32_t bits[2 * MAX_LEVELS];
};

static GridTable grid_table(const ntc_desc* d) {
    GridTable t{};
    const int L = ntc_num_levels(d);
    t.n = 2 * L;
    int64_t off = 0;
    for (int j = 0; j < L; ++j) {
        int32_t a, b;
        level_res(d, j, &a, &b);
        t.start[2 * j] = off;
        t.bits[2 * j] = d->b0;
        off += (int64_t)a * a * d->c0;
        t.start[2 * j + 1] = off;
        t.bits[2 * j + 1] = d->b1;
        off += (int64_t)b * b * d->c1;
    }
    t.start[2 * L] = off;
    return t;
}

// idx = floor(v N + 1/2) computed without the fp32 rounding of (vN + 1/2): t = vN is exact,
// f = floor(t), t - f is exact, then round half up (R9).
__global__ void quantize_kernel(const float* __restrict__ lat, uint8_t* __restrict__ codes, const GridTable t) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= t.start[t.n]) return;
    int g = 0;
    while (i >= t.start[g + 1]) ++g;
    const int B = t.bits[g];
    const int N = 1 << B;
    const float v = lat[i] * (float)N;
    const float f = floorf(v);
    float idx = f + ((v - f) >= 0.5f ? 1.0f : 0.0f);
    idx = fminf(fmaxf(idx, (float)(-(N / 2 - 1))), (float)(N / 2));
    codes[i] = (uint8_t)((int)idx + N / 2 - 1);
}

extern "C" ntc_status ntc_quantize_latents(const ntc_desc* d, const float* latents, uint8_t* codes,
                                           ntc_stream stream) {
    if (ntc_status s = check_desc(d)) return s;
    if (!latents || !codes) return fail(NTC_ERR_INVALID_ARGUMENT, "NULL buffer");
    const GridTable t = grid_table(d);
    const int64_t n = t.start[t.n];
    quantize_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(latents, codes, t);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? NTC_OK : cuda_fail(e, "quantize_kernel");
}

__global__ void dequantize_kernel(const uint8_t* __restrict__ codes, float* __restrict__ lat, const GridTable t) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= t.start[t.n]) return;
    int g = 0;
    while (i >= t.start[g + 1]) ++g;
    const int N = 1 << t.bits[g];
    lat[i] = (float)((int)codes[i] - (N / 2 - 1)) / (float)N;
}

extern "C" ntc_status ntc_dequantize_codes(const ntc_desc* d, const uint8_t* codes, float* latents,
                                           ntc_stream stream) {
    if (ntc_status s = check_desc(d)) return s;
    if (!latents || !codes) return fail(NTC_ERR_INVALID_ARGUMENT, "NULL buffer");
    const GridTable t = grid_table(d);
    const int64_t n = t.start[t.n];
    dequantize_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(codes, latents, t);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? NTC_OK : cuda_fail(e, "dequantize_kernel");
}

// ------------------------------------------------------------------ material
#include "material.h"

// pack C codes (B bits each, LSB first) of one cell into CELL bytes
__global__ void pack_kernel(const uint8_t* __restrict__ codes, int64_t src_off, int64_t ncells, int C, int B,
                            int cell_bytes, uint8_t* __restrict__ dst) {
    const int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (cell >= ncells) return;
    uint32_t w[4] = {0, 0, 0, 0};
    const uint8_t* src = codes + src_off + cell * C;
    for (int ch = 0; ch < C; ++ch) {
        const int bit = ch * B;
        w[bit >> 5] |= ((uint32_t)src[ch] & ((1u << B) - 1u)) << (bit & 31);
    }
    uint8_t* o = dst + cell * cell_bytes;
    for (int b = 0; b < cell_bytes; ++b) o[b] = (uint8_t)(w[b >> 2] >> (8 * (b & 3)));
}

static uint16_t float_to_half_bits(double v) {
    __half_raw r = __half(__double2half(v));
    return r.x;
}

extern "C" ntc_status ntc_material_create(const ntc_desc* d, const uint8_t* codes, const uint16_t* weights_f16,
                                          ntc_stream stream, ntc_material** out) {
    if (ntc_status s = check_desc(d)) return s;
    if (!codes || !weights_f16 || !out) return fail(NTC_ERR_INVALID_ARGUMENT, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    auto* m = new ntc_material();
    m->d = *d;
    m->pid = profile_id(d);
    m->M = ntc_num_mips(d);
    m->L = ntc_num_levels(d);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, dev);
    const int cb0 = pow2_bytes(d->c0 * d->b0), cb1 = pow2_bytes(d->c1 * d->b1);
    // packed grid layout (each grid 16-byte aligned)
    int64_t bytes = 0;
    std::vector<int64_t> src_off(2 * m->L), ncell(2 * m->L);
    for (int j = 0; j < m->L; ++j) {
        int32_t r0, r1;
        int64_t o0, o1;
        ntc_grid_layout(d, j, &r0, &r1, &o0, &o1);
        m->lv[j].r0 = r0;
        m->lv[j].r1 = r1;
        m->lv[j].lr0 = ilog2i(r0);
        m->lv[j].lr1 = ilog2i(r1);
        m->lv[j].off0 = bytes;
        bytes += ((int64_t)r0 * r0 * cb0 + 15) / 16 * 16;
        m->lv[j].off1 = bytes;
        bytes += ((int64_t)r1 * r1 * cb1 + 15) / 16 * 16;
        src_off[2 * j] = o0;
        src_off[2 * j + 1] = o1;
        ncell[2 * j] = (int64_t)r0 * r0;
        ncell[2 * j + 1] = (int64_t)r1 * r1;
    }
    const int hm = d->hidden_mats;
    m->wimg_bytes = decode_wimg_bytes(m->pid, hm);
    cudaError_t e = cudaMalloc(&m->grids, bytes + 16);
    if (e == cudaSuccess) e = cudaMalloc(&m->wimg, m->wimg_bytes);
    if (e != cudaSuccess) {
        ntc_material_destroy(m);
        return cuda_fail(e, "cudaMalloc(material)");
    }
    cudaMemsetAsync(m->grids, 0, bytes + 16, st);
    cudaMemsetAsync(m->wimg, 0, m->wimg_bytes, st);
    for (int j = 0; j < m->L; ++j)
        for (int k = 0; k < 2; ++k) {
            const int64_t n = ncell[2 * j + k];
            pack_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
                codes, src_off[2 * j + k], n, k ? d->c1 : d->c0, k ? d->b1 : d->b0, k ? cb1 : cb0,
                m->grids + (k ? m->lv[j].off1 : m->lv[j].off0));
        }
    e = build_wimg(m->pid, hm, weights_f16, d->channels, reinterpret_cast<uint8_t*>(m->wimg), st);
    // the output bias b3 (last c parameters) travels as a kernel parameter
    uint16_t hb3[16] = {0};
    const int64_t P = ntc_num_params(d);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(hb3, weights_f16 + P - d->channels, sizeof(uint16_t) * d->channels,
                            cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    for (int i = 0; i < 16; ++i) {
        __half_raw r;
        r.x = i < d->channels ? hb3[i] : 0;
        m->b3[i] = __half2float(__half(r));
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) {
        ntc_material_destroy(m);
        return cuda_fail(e, "material upload");
    }
    *out = m;
    return NTC_OK;
}

extern "C" void ntc_material_destroy(ntc_material* m) {
    if (!m) return;
    if (m->grids) cudaFree(m->grids);
    if (m->wimg) cudaFree(m->wimg);
    delete m;
}

// ------------------------------------------------------------------ decode
static double tri_wave(double t) { return 4.0 * std::fabs((t - std::floor(t)) - 0.5) - 1.0; }

namespace ntc {
uint16_t host_f16(double v) { return float_to_half_bits(v); }
double host_tri(double t) { return tri_wave(t); }
}  // namespace ntc

namespace ntc {
DecodeParams base_params(const ntc_material* m);
cudaError_t decode_queries(const ntc_material* m, const ntc_query* q, int64_t n, uint16_t* out, int32_t* status,
                           cudaStream_t s);
}  // namespace ntc

DecodeParams ntc::base_params(const ntc_material* m) {
    DecodeParams p;
    memset(&p, 0, sizeof p);
    p.grids = m->grids;
    p.wimg = m->wimg;
    p.wimg_bytes = m->wimg_bytes;
    p.W = m->d.width;
    p.c = m->d.channels;
    p.act = m->d.activation;
    p.M = m->M;
    p.L = m->L;
    for (int j = 0; j < m->L; ++j) p.lv[j] = m->lv[j];
    memcpy(p.b3, m->b3, sizeof p.b3);
    for (int mi = 0; mi < m->M; ++mi) {
        p.level_of[mi] = (int8_t)ntc_level_of_mip(&m->d, mi);
        const double lod = m->M > 1 ? (double)mi / (double)(m->M - 1) : 0.0;  // R6
        p.lod_word[mi] = (uint32_t)float_to_half_bits(lod) | ((uint32_t)float_to_half_bits(1.0) << 16);
    }
    // tiled triangle-wave PE (R5): per axis, octaves h = 0..2, phases 0 and 1/4
    for (int q = 0; q < 8; ++q) {
        uint16_t v[6];
        for (int h = 0; h < 3; ++h) {
            const double t = (double)(1 << h) * q / 8.0;
            v[2 * h] = float_to_half_bits(tri_wave(t));
            v[2 * h + 1] = float_to_half_bits(tri_wave(t - 0.25));
        }
        for (int k = 0; k < 3; ++k) p.pe_words[q][k] = (uint32_t)v[2 * k] | ((uint32_t)v[2 * k + 1] << 16);
        p.pe_words[q][3] = 0;
    }
    return p;
}

static int grid_for(const ntc_material* m, int64_t tiles) {
    int64_t g = (tiles + NWG - 1) / NWG;
    if (g > m->num_sms) g = m->num_sms;
    return (int)(g < 1 ? 1 : g);
}

static ntc_status launch_tiles(const ntc_material* m, int mip_first, int mip_count, uint16_t* out,
                               const int64_t* out_off, const int64_t* row_stride, cudaStream_t st, int part = 0,
                               int nparts = 1) {
    DecodeParams p = base_params(m);
    p.mode = 0;
    p.out = out;
    p.mip_first = mip_first;
    p.mip_count = mip_count;
    int64_t t = 0;
    for (int i = 0; i < mip_count; ++i) {
        const int64_t w = m->d.width >> (mip_first + i);
        p.tile_start[i] = (int32_t)t;
        t += (w * w + TILE_M - 1) / TILE_M;
        p.out_off[i] = out_off[i];
        p.row_stride[i] = row_stride[i];
    }
    for (int i = mip_count; i <= MAX_MIPS; ++i) p.tile_start[i] = INT32_MAX;
    p.tile_start[mip_count] = (int32_t)t;
    p.n_tiles = (int32_t)t;
    p.lin_tiles = 0;
    for (int i = 0; i < mip_count; ++i) {
        const int64_t w = m->d.width >> (mip_first + i);
        if ((w * w) % TILE_M || out_off[i] != (int64_t)p.tile_start[i] * TILE_M * m->d.channels ||
            row_stride[i] != w * m->d.channels)
            break;
        p.lin_tiles = p.tile_start[i + 1];
    }
    p.tma_tiles = ((uintptr_t)out & 15) == 0 ? p.lin_tiles : 0;
    p.pair_tiles = 0;
    if ((m->d.channels & 1) && ((uintptr_t)out & 3) == 0)
        for (int i = 0; i < mip_count; ++i) {
            if ((m->d.width >> (mip_first + i)) < TILE_M || (out_off[i] & 1) || (row_stride[i] & 1)) break;
            p.pair_tiles = p.tile_start[i + 1];
        }
    // part of the tile range: [t*part/nparts, t*(part+1)/nparts)
    const int64_t t0 = t * part / nparts, t1 = t * (part + 1) / nparts;
    p.tile_first = (int32_t)t0;
    p.n_tiles = (int32_t)t1;
    if (t1 <= t0) return NTC_OK;
    cudaError_t e = launch_decode(m->pid, m->d.hidden_mats, p, grid_for(m, t1 - t0), st);
    return e == cudaSuccess ? NTC_OK : cuda_fail(e, "decode_kernel");
}

extern "C" ntc_status ntc_decode_chain(const ntc_material* m, uint16_t* out, ntc_stream stream) {
    if (!m || !out) return fail(NTC_ERR_INVALID_ARGUMENT, "NULL argument");
    int64_t off[MAX_MIPS], rs[MAX_MIPS];
    for (int mi = 0; mi < m->M; ++mi) {
        off[mi] = ntc_mip_offset(&m->d, mi) * m->d.channels;
        rs[mi] = (int64_t)(m->d.width >> mi) * m->d.channels;
    }
    return launch_tiles(m, 0, m->M, out, off, rs, (cudaStream_t)stream);
}

extern "C" ntc_status ntc_decode_chain_part(const ntc_material* m, int32_t part, int32_t nparts, uint16_t* out,
                                            ntc_stream stream) {
    if (!m || !out) return fail(NTC_ERR_INVALID_ARGUMENT, "NULL argument");
    if (nparts < 1 || part < 0 || part >= nparts) return fail(NTC_ERR_INVALID_ARGUMENT, "bad part/nparts");
    int64_t off[MAX_MIPS], rs[MAX_MIPS];
    for (int mi = 0; mi < m->M; ++mi) {
        off[mi] = ntc_mip_offset(&m->d, mi) * m->d.channels;
        rs[mi] = (int64_t)(m->d.width >> mi) * m->d.channels;
    }
    return launch_tiles(m, 0, m->M, out, off, rs, (cudaStream_t)stream, part, nparts);
}

extern "C" ntc_status ntc_decode_mip(const ntc_material* m, int32_t mip, uint16_t* out, int64_t row_stride_elems,
                                     ntc_stream stream) {
    if (!m || !out) return fail(NTC_ERR_INVALID_ARGUMENT, "NULL argument");
    if (mip < 0 || mip >= m->M) return fail(NTC_ERR_INVALID_ARGUMENT, "mip %d out of range [0,%d)", mip, m->M);
    if (row_stride_elems < (int64_t)(m->d.width >> mip) * m->d.channels)
        return fail(NTC_ERR_INVALID_ARGUMENT, "row stride too small");
    int64_t off = 0;
    return launch_tiles(m, mip, 1, out, &off, &row_stride_elems, (cudaStream_t)stream);
}

cudaError_t ntc::decode_queries(const ntc_material* m, const ntc_query* q, int64_t n, uint16_t* out, int32_t* status,
                                cudaStream_t s) {
    DecodeParams p = base_params(m);
    p.mode = 1;
    p.q = q;
    p.nq = n;
    p.out = out;
    p.status = status;
    p.pair_tiles = (m->d.channels & 1) && ((uintptr_t)out & 3) == 0 ? (int32_t)(n / TILE_M) : 0;
    return launch_decode(m->pid, m->d.hidden_mats, p, grid_for(m, (n + TILE_M - 1) / TILE_M), s);
}

extern "C" ntc_status ntc_decode_texels(const ntc_material* m, const ntc_query* q, int64_t n, uint16_t* out,
                                        int32_t* status, ntc_stream stream) {
    if (!m) return fail(NTC_ERR_INVALID_ARGUMENT, "NULL material");
    if (n < 0) return fail(NTC_ERR_INVALID_ARGUMENT, "n < 0");
    if (n == 0) return NTC_OK;
    if (!q || !out) return fail(NTC_ERR_INVALID_ARGUMENT, "NULL buffer");
    cudaError_t e = decode_queries(m, q, n, out, status, (cudaStream_t)stream);
    return e == cudaSuccess ? NTC_OK : cuda_fail(e, "decode_kernel(queries)");
}

extern "C" ntc_status ntc_debug_assemble(const ntc_material* m, const ntc_query* q, int64_t n, int32_t* addr,
                                         uint16_t* X, ntc_stream stream) {
    if (!m || !q || !addr || !X || n < 0) return fail(NTC_ERR_INVALID_ARGUMENT, "bad argument");
    if (n == 0) return NTC_OK;
    DecodeParams p = base_params(m);
    p.mode = 2;
    p.q = q;
    p.nq = n;
    p.dbg_addr = addr;
    p.dbg_X = X;
    cudaError_t e = launch_debug_assemble(m->pid, p, (cudaStream_t)stream);
    return e == cudaSuccess ? NTC_OK : cuda_fail(e, "debug_assemble_kernel");
}
