/*
 * ntc_oracle.h -- CPU ORACLE FOR TESTS ONLY (test infrastructure, not product code).
 *
 * A plain, slow, scalar fp64 C implementation of what the NTC hot path computes
 * (Vaidyanathan et al., "Random-Access Neural Compression of Material Textures",
 * arXiv 2305.17105; text in /root/reference/PAPER.md, cited here as PAPER.md:<line>).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The CUDA product path (paper_2305_17105_b200/) shares
 * no code, header, table or constant generator with it, and never calls it.
 *
 * Every function follows the paper's definition step by step, in its order and
 * notation; where the paper is silent the reading taken is the one listed in
 * DESIGN.md "Readings" (numbered R1..R25 there, mirrored in comments below).
 *
 * Parity status per function:
 *   geometry / level mapping / quantisation / PE / hardGELU / Philox / MLP /
 *   gradients (finite differences) / Adam (closed-form single step) : pinned.
 *   end-to-end decode value : composition of pinned parts (the paper prints no
 *   worked decode example) -- pinned through an independent fp64 numpy
 *   re-derivation test of the composition on tiny grids.
 */
#ifndef NTC_ORACLE_H
#define NTC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* A material's shape: texture set w x h x c + profile (Table 2,
 * PAPER.md:674-688) + MLP depth/activation. w == h. */
typedef struct {
    int32_t width;        /* W = H, power of two >= 4                          */
    int32_t channels;     /* c, output channels, 1..16                          */
    int32_t g0_ratio;     /* G^0_0 resolution = W / g0_ratio (Table 2)          */
    int32_t c0, b0;       /* G_0 channels C_0 and bits B_0                      */
    int32_t c1, b1;       /* G_1 channels C_1 and bits B_1                      */
    int32_t hidden_mats;  /* 1: [D,64,64,c]  2: [D,64,64,64,c]  (R11)           */
    int32_t activation;   /* 0: hardGELU, 1: exact GELU */
} ntco_desc;

/* ---- geometry / addressing (Table 1) ---- */
int32_t ntco_num_mips(int32_t width);
int32_t ntco_num_levels(const ntco_desc* d);
int32_t ntco_level_of_mip(const ntco_desc* d, int32_t mip);
void    ntco_grid_res(const ntco_desc* d, int32_t level, int32_t* r0, int32_t* r1);
int64_t ntco_grid_offset(const ntco_desc* d, int32_t level, int32_t k);  /* latent/code offset */
int64_t ntco_num_latents(const ntco_desc* d);
int32_t ntco_input_dim(const ntco_desc* d);                              /* D = 4C0+C1+12+1 */
int64_t ntco_num_params(const ntco_desc* d);
/* taps: out_i[0]=level, out_i[1..8] = G0 taps (x,y)x4, out_i[9..16] = G1 taps (x,y)x4;
 * out_w[0..3] = bilinear weights of the G1 taps.                                   */
void    ntco_address(const ntco_desc* d, int32_t mip, int32_t x, int32_t y,
                     int32_t out_i[17], double out_w[4]);

/* ---- scalar quantisation ---- */
int32_t ntco_quantize(double v, int32_t bits);        /* -> code in [0, 2^B - 1] */
double  ntco_dequantize(int32_t code, int32_t bits);  /* -> idx * Q              */
double  ntco_quant_lo(int32_t bits);
double  ntco_quant_hi(int32_t bits);
void    ntco_quantize_latents(const ntco_desc* d, const float* latents, uint8_t* codes);

/* ---- inputs ---- */
double   ntco_tri(double t);
void     ntco_pe(int32_t x, int32_t y, double out[12]);
uint16_t ntco_f64_to_f16(double v);       /* IEEE binary16, round to nearest even */
double   ntco_f16_to_f64(uint16_t h);
uint16_t ntco_lod_f16(int32_t mip, int32_t num_mips);
/* X as fp16 bit patterns (D values), from quantised codes. */
void     ntco_assemble(const ntco_desc* d, const uint8_t* codes, int32_t mip,
                       int32_t x, int32_t y, uint16_t* X);

/* ---- network ---- */
double ntco_hardgelu(double x);
double ntco_hardgelu_grad(double x);
double ntco_gelu(double x);      /* exact GELU, activation = 1 */
double ntco_gelu_grad(double x);
/* params in ABI order (W1[64][D], b1[64], W2[64][64], b2[64], [W2b, b2b], W3[c][64], b3[c]) */
void   ntco_mlp_forward(const ntco_desc* d, const double* params, const double* X, double* y);

/* ---- decode (Fig 3) ---- */
/* queries: int32 triples (x, y, mip); out: n x c doubles, clamped to [0,1] (R13). */
void ntco_decode_texels(const ntco_desc* d, const uint8_t* codes, const uint16_t* weights_f16,
                        const int32_t* queries, int64_t n, double* out, int32_t nthreads);
void ntco_decode_mip(const ntco_desc* d, const uint8_t* codes, const uint16_t* weights_f16,
                     int32_t mip, double* out, int32_t nthreads);

/* ---- filtering on top of random-access decode ----
 * uvl: n x (u, v, lod) doubles, u, v in [0,1) texture coordinates, lod >= 0.
 * mode 0 nearest (mip floor(lod+1/2)), 1 bilinear (4 decodes), 2 trilinear (8 decodes),
 * 3 stochastic bilinear (U(-1/2,1/2) texel jitter, 1 decode), 4 stochastic trilinear
 * (+ U(-1/2,1/2) LOD jitter).  Jitter: Philox4x32-10 key = seed, ctr = (i, i>>32, 0,
 * 'FILT'), words 0/1/2 -> (2(w>>9)+1) 2^-24 - 1/2.  out: n x c doubles.                 */
void ntco_filter(const ntco_desc* d, const uint8_t* codes, const uint16_t* weights_f16, const double* uvl,
                 int64_t n, int32_t mode, uint64_t seed, double* out, int32_t nthreads);

/* ---- training ---- */
void   ntco_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
double ntco_noise(uint64_t seed, uint32_t step, int64_t latent_index, int32_t bits);
/* crops: n_crops x (x0, y0, w, h) at mip `mip`; ref_f16: mip image (h_m x w_m x c) fp16.
 * round_f16 = 1 is the definition (X and W in the fp16 network-input format, R14);
 * round_f16 = 0 skips those two roundings (exact fp64, for finite-difference checks only).
 * Returns the mean-L2 loss; writes dparams[P] and dlatents[num_latents] (dense; overwritten). */
double ntco_train_grads(const ntco_desc* d, const float* latents, const float* params_f32,
                        int32_t mip, int32_t n_crops, const int32_t* crops,
                        const uint16_t* ref_f16, uint64_t seed, uint32_t step, int32_t noise_on,
                        int32_t round_f16, double* dparams, double* dlatents, int32_t nthreads);
/* One Adam step on n fp32 parameters (state updated in place); sparse: skip g == 0;
 * clamp_on: clamp to [lo, hi] after the update. */
void   ntco_adam(int64_t n, float* p, float* m, float* v, const float* g, int32_t t,
                 double lr, double beta1, double beta2, double eps, int32_t sparse,
                 int32_t clamp_on, double lo, double hi);

#ifdef __cplusplus
}
#endif
#endif
