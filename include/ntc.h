/*
 * ntc.h -- C ABI of the B200 (sm_100a) Neural Texture Compression hot path.
 *
 * Method: Vaidyanathan et al., "Random-Access Neural Compression of Material
 * Textures" (arXiv 2305.17105).  Citations are PAPER.md:<line> (the paper's text) and
 * DESIGN.md R<n> (the readings taken where the paper is silent).
 *
 * Conventions (all entry points):
 *  - Plain C types only.  Pointers documented "device" are CUDA device pointers owned
 *    by the caller (e.g. torch tensors); pointers documented "host" are host memory.
 *  - Hot-path calls (ntc_decode_*, ntc_train_step, ntc_debug_assemble) enqueue work on
 *    `stream` (a cudaStream_t, 0 = legacy default stream), allocate nothing, never
 *    synchronise the host, and return NTC_OK once the work is enqueued.
 *  - Host-checkable argument errors return NTC_ERR_INVALID_ARGUMENT / NTC_ERR_UNSUPPORTED
 *    synchronously and enqueue nothing.  Launch failures return NTC_ERR_CUDA.
 *    ntc_last_error() returns a thread-local message for the last failing call.
 *  - Device-detected errors (an out-of-range query, a non-finite loss) are OR-ed into a
 *    caller-owned int32 device status word; the rest of the batch completes normally.
 *  - Only ntc_material_create / ntc_trainer_create allocate (and their _destroy free).
 */
#ifndef NTC_H
#define NTC_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* ntc_stream; /* == cudaStream_t */

typedef enum {
    NTC_OK = 0,
    NTC_ERR_INVALID_ARGUMENT = 1,
    NTC_ERR_OUT_OF_RANGE = 2, /* device status bit: a query had x/y/mip out of range   */
    NTC_ERR_DATA = 3,
    NTC_ERR_NONFINITE = 4,    /* device status bit: non-finite loss       */
    NTC_ERR_CUDA = 5,
    NTC_ERR_UNSUPPORTED = 6   /* profile / depth not compiled into this library         */
} ntc_status;

/* A material: texture set w x h x c (w == h, power of two >= 4, c <= 16),
 * feature-grid profile (Table 2: G^0_0 = W/g0_ratio, C_k x B_k) and the
 * decoder MLP [D, 64, 64, c] (hidden_mats = 1) or [D, 64, 64, 64, c]
 * (hidden_mats = 2, reading R11), D = 4C0 + C1 + 12 + 1, hardGELU
 * (activation = 0) or exact GELU x Phi(x) (activation = 1, PAPER.md:496;
 * decode and training).  Compiled profiles: NTC 0.2/0.5/1.0/2.25, depth 1 or 2.           */
typedef struct {
    int32_t width;
    int32_t channels;
    int32_t g0_ratio;
    int32_t c0, b0;
    int32_t c1, b1;
    int32_t hidden_mats;
    int32_t activation;
} ntc_desc;

/* One random-access query (8 bytes): texel (x, y) of mip `mip`; `material` indexes the
 * material array of ntc_decode_texels_multi (ignored by the single-material calls). */
typedef struct {
    uint16_t x, y;
    uint8_t mip;
    uint8_t material;
    uint8_t pad[2];
} ntc_query;

const char* ntc_last_error(void);

/* ---------------------------------------------------------------- geometry (host, pure)
 * Mip chain down to 1x1 (Table 1).  Feature levels: levels continue while
 * G1 is >= 1x1, up to ceil((M-3)/2) levels for M mips; mips 0-3 -> level 0, then pairs, the
 * last level takes the bottom 2-3 mips (R7); r0 = W/ratio/4^j, r1 = r0/2 (Table 1, R8).  Latents/codes of all grids live in one
 * canonical array: grids [F0.G0, F0.G1, F1.G0, ...], each (y, x, ch) row-major.            */
int32_t ntc_num_mips(const ntc_desc* d);
int32_t ntc_num_levels(const ntc_desc* d);
int32_t ntc_level_of_mip(const ntc_desc* d, int32_t mip);
/* r0/r1: grid resolutions of level j; off0/off1: element offsets of G0/G1 in the canonical array. */
ntc_status ntc_grid_layout(const ntc_desc* d, int32_t level, int32_t* r0, int32_t* r1, int64_t* off0,
                           int64_t* off1);
int64_t ntc_num_latents(const ntc_desc* d);
int64_t ntc_num_params(const ntc_desc* d); /* P, parameters in ABI order (below) */
int64_t ntc_chain_texels(const ntc_desc* d); /* sum over mips of w_m^2 */
int64_t ntc_mip_offset(const ntc_desc* d, int32_t mip); /* texel offset of mip in a dense chain */

/* ---------------------------------------------------------------- quantisation (a0)
 * codes[i] = clamp(floor(latents[i]/Q + 1/2), -(N/2-1), N/2) + N/2 - 1 with N = 2^B, Q = 1/N,
 * B = b0 for G0 grids, b1 for G1 grids (R9, R10).  Bit-exact.
 * latents: device fp32 [num_latents]; codes: device uint8 [num_latents].                  */
ntc_status ntc_quantize_latents(const ntc_desc* d, const float* latents, uint8_t* codes, ntc_stream stream);
/* latents[i] = (codes[i] - (N/2 - 1)) Q: the bin centres.  Used to freeze the
 * explicitly quantised latents for the weight-only finetune.               */
ntc_status ntc_dequantize_codes(const ntc_desc* d, const uint8_t* codes, float* latents, ntc_stream stream);

/* ---------------------------------------------------------------- material (decode side)
 * codes: device uint8 [num_latents], canonical layout, each < 2^B of its grid.
 * weights_f16: device uint16 [P] fp16 bit patterns, ABI order:
 *   W1[64][D], b1[64], W2[64][64], b2[64], (hidden_mats == 2: W2b[64][64], b2b[64]),
 *   W3[c][64], b3[c]   (row-major [out][in]).
 * Creates the device-resident material: bit-packed grids + UMMA-swizzled fp16 weight image.
 * Synchronises `stream` once (the material is ready on return).  Caller keeps ownership of
 * its inputs; the library owns *out until ntc_material_destroy.                           */
typedef struct ntc_material ntc_material;
ntc_status ntc_material_create(const ntc_desc* d, const uint8_t* codes, const uint16_t* weights_f16,
                               ntc_stream stream, ntc_material** out);
void ntc_material_destroy(ntc_material* m);

/* ---------------------------------------------------------------- decode (a1..a7)
 * Per texel: level select, 2x2 unfiltered G0 gather + bilinear G1,
 * tiled triangle-wave PE + LOD, MLP with hardGELU, no output
 * activation, clamp to [0,1] and fp16 store (R13).
 *
 * ntc_decode_texels: q device [n] queries (any mips, any order); out device fp16 [n][c].
 *   A query with x or y >= w_m or mip >= M sets NTC_ERR_OUT_OF_RANGE in *status (device
 *   int32, may be NULL) and writes NaN to its row.  n == 0 is a no-op.
 * ntc_decode_mip: out device fp16, row y at out + y*row_stride_elems, texel x at +x*c;
 *   row_stride_elems >= w_m*c.  mip >= M -> NTC_ERR_INVALID_ARGUMENT.
 * ntc_decode_chain: every mip in one launch, dense (y, x, ch) per mip, mips concatenated
 *   (mip m starts at texel ntc_mip_offset(m)); out device fp16 [chain_texels][c].          */
ntc_status ntc_decode_texels(const ntc_material* m, const ntc_query* q, int64_t n, uint16_t* out,
                             int32_t* status, ntc_stream stream);
ntc_status ntc_decode_mip(const ntc_material* m, int32_t mip, uint16_t* out, int64_t row_stride_elems,
                          ntc_stream stream);
ntc_status ntc_decode_chain(const ntc_material* m, uint16_t* out, ntc_stream stream);
/* Multi-GPU partition of ntc_decode_chain (multi-GPU): the chain's 128-texel tiles
 * are split into nparts contiguous ranges of equal size; this call decodes range `part`
 * into the same chain layout as ntc_decode_chain (other texels of out are not written).  */
ntc_status ntc_decode_chain_part(const ntc_material* m, int32_t part, int32_t nparts, uint16_t* out,
                                 ntc_stream stream);

/* Multi-material random-access decode (the B200 analog of the paper's
 * divergence handling for neighbouring pixels of different materials):
 * queries of up to NTC_MAX_MATERIALS materials in one call.  The library buckets the queries
 * by q[i].material on the device (count, scan, scatter into scratch), then one persistent
 * launch walks the material-sorted tile list; every 128-texel tile has a single weight set,
 * which a CTA swaps in SMEM only when its share of the list crosses a material boundary.
 * mats: host array [n_mats] of materials that all share one ntc_desc (same dimensions,
 * profile, channels and depth; else NTC_ERR_INVALID_ARGUMENT).  q: device [n] queries;
 * out: device fp16 [n][c], row i for query i (input order).  A query whose material index is
 * >= n_mats, or whose texel is out of range, gets a NaN row and sets NTC_ERR_OUT_OF_RANGE in
 * *status (device int32, may be NULL).  scratch: device, >= ntc_decode_multi_scratch_bytes(n)
 * bytes, 16-byte aligned, owned by the caller.  n <= 2^31 - 1.                           */
#define NTC_MAX_MATERIALS 256
int64_t ntc_decode_multi_scratch_bytes(int64_t n);
ntc_status ntc_decode_texels_multi(const ntc_material* const* mats, int32_t n_mats, const ntc_query* q, int64_t n,
                                   uint16_t* out, int32_t* status, void* scratch, int64_t scratch_bytes,
                                   ntc_stream stream);

/* Texture filtering on top of random-access decode.
 * uvl: device fp32 [n][3] = (u, v, lod): u, v in [0,1) (texel x of mip m has centre
 * (x + 1/2)/w_m), lod >= 0.  mode:
 *   0 nearest: mip floor(lod + 1/2), texel floor(u w_m) (clamped);
 *   1 bilinear: 4 decodes at mip floor(lod + 1/2), clamp-to-edge;
 *   2 trilinear: 8 decodes, mips floor(lod) and floor(lod)+1 blended by frac(lod);
 *   3 stochastic bilinear: (u, v) jittered by U(-1/2, 1/2) texel, then nearest -- 1 decode
 *     (PAPER.md:631-633); 4 stochastic trilinear: LOD jittered by U(-1/2, 1/2) too.
 *   Jitter: Philox4x32-10, key = seed, ctr = (i, i >> 32, 0, 'FILT'), words 0/1/2 ->
 *   (2(w >> 9) + 1) 2^-24 - 1/2.
 * out: device fp16 [n][c]; scratch: device, ntc_filter_scratch_bytes(n, mode, c) bytes
 * (query list, blend weights, tap decodes).  Each decode is clamped to [0,1] (R13).       */
int64_t ntc_filter_scratch_bytes(int64_t n, int32_t mode, int32_t channels);
ntc_status ntc_filter_texels(const ntc_material* m, const float* uvl, int64_t n, int32_t mode, uint64_t seed,
                             uint16_t* out, void* scratch, ntc_stream stream);

/* Tests only: runs the decode kernels' own addressing + input assembly for n queries and
 * writes addr device int32 [n][17] = {level, G0 taps (x,y) x4, G1 taps (x,y) x4} and
 * X device uint16 [n][D] (fp16 network input, R4).  Out-of-range queries are
 * clamped to mip M-1, texel (0,0).                                                        */
ntc_status ntc_debug_assemble(const ntc_material* m, const ntc_query* q, int64_t n, int32_t* addr,
                              uint16_t* X, ntc_stream stream);

/* ---------------------------------------------------------------- training (t1..t8)
 * Autodecoder step: latents and MLP weights optimised
 * jointly with Adam on the mean L2 loss over B*c values (R17); simulated quantisation by
 * U(-Q/2, Q/2) noise, one draw per latent per step (R16: Philox4x32-10,
 * key = seed, counter = (i/4, i/2^34, step, 'NOIS'), word i%4, u = (2(w>>9)+1) 2^-24);
 * latents clamped to [-(N-1)Q/2, NQ/2] after each update.
 *
 * All buffers are caller-owned device fp32 arrays in the canonical layouts:
 *   latents/m_lat/v_lat/grad_lat/noisy [num_latents], params/m_par/v_par/grad_par [P]. */
typedef struct {
    float *latents, *m_lat, *v_lat, *grad_lat;
    float *params, *m_par, *v_par, *grad_par;
    float* noisy; /* scratch (>= 2*num_latents bytes): fp16 noisy latents, written inside the
                   * batch footprint only                                                   */
} ntc_train_buffers;

/* One batch = n_crops crops at one mip: crops host int32 [n_crops][4] =
 * (x0, y0, w, h), each inside the mip; ref device fp16 reference mip image, 4-byte
 * aligned (else NTC_ERR_INVALID_ARGUMENT), row y at ref + y*ref_row_stride_elems (R24).
 * n_crops <= NTC_MAX_CROPS.
 * norm_texels: the B of the mean over B*c values (R17); 0 = this batch's own texel count.
 * A data-parallel rank passes the global batch's count so that the sum of the ranks'
 * gradients is the global gradient.                                                     */
#define NTC_MAX_CROPS 64
typedef struct {
    int32_t mip;
    int32_t n_crops;
    const int32_t* crops;
    const uint16_t* ref;
    int64_t ref_row_stride_elems;
    int64_t norm_texels;
} ntc_batch;

typedef struct {
    float lr_latent, lr_weight; /* PAPER.md:575 (0.01 / 0.005 initial, cosine by the caller) */
    float beta1, beta2, eps;    /* R18: 0.9 / 0.999 / 1e-8                                   */
    int32_t step;               /* Adam t (>= 1) and the noise counter                        */
    uint64_t seed;
    int32_t noise_on;           /* 1: simulated quantisation noise             */
    int32_t dense_latent_adam;  /* 0: footprint-sparse Adam, skip g == 0 (R18); 1: dense      */
    int32_t freeze_latents;     /* 1: frozen phase: latents are held at their
                                 * quantised values -- GRADS skips the latent-gradient scatter,
                                 * APPLY updates only the weights; use with noise_on = 0      */
} ntc_train_hparams;

enum { NTC_STEP_GRADS = 1, NTC_STEP_APPLY = 2 };

/* Training scratch (per-CTA partial weight gradients, loss partials); sized for d. */
typedef struct ntc_trainer ntc_trainer;
ntc_status ntc_trainer_create(const ntc_desc* d, ntc_trainer** out);
void ntc_trainer_destroy(ntc_trainer* t);

/* flags & NTC_STEP_GRADS: zero grad_par and grad_lat inside the batch footprint, write noisy
 *   latents there, run the fused forward+backward, write grad_par, scatter grad_lat, and
 *   write the batch loss to *loss (device fp32).  Non-finite loss -> NTC_ERR_NONFINITE in
 *   *status (device int32, may be NULL).
 * flags & NTC_STEP_APPLY: Adam on params (dense) and on latents (footprint-sparse unless
 *   dense_latent_adam), then the latent clamp.  Between the two phases the caller may
 *   all-reduce grad_par / grad_lat across data-parallel ranks (multi-GPU).
 *   APPLY uses this batch's footprint; ntc_train_footprint describes it.                  */
ntc_status ntc_train_step(ntc_trainer* t, const ntc_desc* d, const ntc_train_buffers* buf,
                          const ntc_batch* batch, const ntc_train_hparams* hp, float* loss, int32_t* status,
                          uint32_t flags, ntc_stream stream);

/* Footprint of a batch (host, pure): disjoint boxes (level, grid k, x0, y0, x1, y1) of
 * inclusive cell ranges that together cover exactly the grid cells read by the crops'
 * texels (at most 256 boxes; a pathological overlap pattern falls back to one bounding box
 * per grid).  Returns the box count (-1 on a bad batch); pass boxes = NULL to query it,
 * otherwise boxes must hold [count][6] int32.                                            */
int32_t ntc_train_footprint(const ntc_desc* d, const ntc_batch* batch, int32_t* boxes);

/* Data-parallel latent-gradient exchange (multi-GPU): the latents inside the
 * footprint of `batch` (normally the GLOBAL batch: every rank's crops) in box order.
 * ntc_footprint_size: element count (host, pure; -1 on a bad batch).
 * ntc_footprint_pack: packed[i] = src[latent of footprint element i] (device fp32).
 * ntc_footprint_unpack: dst[latent of footprint element i] = packed[i], or 0 if packed is
 *   NULL (zeroes the footprint).                                                          */
int64_t ntc_footprint_size(const ntc_desc* d, const ntc_batch* batch);
ntc_status ntc_footprint_pack(const ntc_desc* d, const ntc_batch* batch, const float* src, float* packed,
                              ntc_stream stream);
ntc_status ntc_footprint_unpack(const ntc_desc* d, const ntc_batch* batch, const float* packed, float* dst,
                                ntc_stream stream);

/* Explicit box lists, for the sharded data-parallel mode (multi-GPU: every rank
 * owns a row band of every latent grid and its Adam state).  boxes: host int32 [n][6] in the
 * ntc_train_footprint format (level, grid k, x0, y0, x1, y1), inclusive and disjoint,
 * n <= 256; a box outside its grid -> NTC_ERR_INVALID_ARGUMENT.
 * ntc_boxes_size: latent count covered (host, pure; -1 on bad boxes).
 * ntc_boxes_copy (device fp32, box order, channel-minor within a cell):
 *   NTC_BOX_PACK   dst[i] = src[latent i]            (dst packed, src canonical)
 *   NTC_BOX_UNPACK dst[latent i] = src[i]            (src packed, dst canonical)
 *   NTC_BOX_ADD    dst[latent i] += src[i]
 *   NTC_BOX_ZERO   dst[latent i] = 0                 (src unused)
 * ntc_train_apply_boxes: the APPLY phase of ntc_train_step (Adam on the weights, then on the
 *   latents inside `boxes`, then the latent clamp) for an explicit box list.              */
enum { NTC_BOX_PACK = 0, NTC_BOX_UNPACK = 1, NTC_BOX_ADD = 2, NTC_BOX_ZERO = 3 };
int64_t ntc_boxes_size(const ntc_desc* d, const int32_t* boxes, int32_t n);
ntc_status ntc_boxes_copy(const ntc_desc* d, const int32_t* boxes, int32_t n, const float* src, float* dst,
                          int32_t mode, ntc_stream stream);
ntc_status ntc_train_apply_boxes(ntc_trainer* t, const ntc_desc* d, const ntc_train_buffers* buf,
                                 const int32_t* boxes, int32_t n, const ntc_train_hparams* hp, ntc_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* NTC_H */
