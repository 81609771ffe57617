/*
 * ntc_oracle.c -- CPU ORACLE FOR TESTS ONLY (test infrastructure, not product code).
 * See ntc_oracle.h for the contract.  Plain scalar fp64 loops, no blocking, no
 * fusion, no SIMD: each function is the paper's definition written out, so it can be
 * checked against PAPER.md by eye.  OpenMP only splits independent texels across
 * threads; every reduction is done afterwards in a fixed serial order.
 */
#include "ntc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define HIDDEN 64 /* "two hidden layers, each of size 64 channels" PAPER.md:492 */

/* ------------------------------------------------------------------------- */
/* Geometry and addressing                                                    */
/* ------------------------------------------------------------------------- */

static int32_t ilog2(int32_t v) { int32_t l = 0; while ((1 << (l + 1)) <= v) ++l; return l; }

/* Mip chain down to 1x1: Table 1 lists mips 0..10 for 1024^2. */
int32_t ntco_num_mips(int32_t width) { return ilog2(width) + 1; }

/* R7: a new level is added while G_1 is still at least 1x1, i.e. while
 * floor((W/ratio)/4^j) >= 2 ("it cannot be further downsampled"), but not
 * past the level that holds the bottom mips: "the last feature level represents the bottom
 * three mip levels", so with M mips (0-3 | pairs | tail of 2-3) there are at
 * most ceil((M-3)/2) levels.  The cap binds only for the ratio-2 profiles at even log2 sizes
 * (e.g. 4096^2 NTC 1.0: 5 levels, mips 10-12 on the last).                 */
int32_t ntco_num_levels(const ntco_desc* d) {
    int32_t L = 0;
    int64_t r0 = d->width / d->g0_ratio;
    while (r0 >= 2) { ++L; r0 /= 4; }
    int32_t M = ntco_num_mips(d->width);
    int32_t Lm = (M - 3 + 1) / 2;
    if (Lm < 1) Lm = 1;
    return L < Lm ? L : Lm;
}

/* R7: "the first feature level must represent all higher resolution mips (levels 0 to 3),
 * and the last feature level represents the bottom three mip levels";
 * "Typically, a feature level represents two mip levels" -> level(m) = floor((m-2)/2). */
int32_t ntco_level_of_mip(const ntco_desc* d, int32_t mip) {
    int32_t L = ntco_num_levels(d);
    if (mip <= 3) return 0;
    int32_t j = (mip - 2) / 2;
    return j < L - 1 ? j : L - 1;
}

/* R8: r0 = W/ratio/4^j (Table 1 columns 2-3, Table 2 column 2), r1 = r0/2. */
void ntco_grid_res(const ntco_desc* d, int32_t level, int32_t* r0, int32_t* r1) {
    int32_t g = d->width / d->g0_ratio;
    for (int32_t j = 0; j < level; ++j) g /= 4;
    *r0 = g;
    *r1 = g / 2 > 1 ? g / 2 : 1;
}

/* Canonical concatenated latent layout (shared by codes and fp32 latents):
 * grids in order [F0.G0, F0.G1, F1.G0, F1.G1, ...], each (y, x, ch) row-major.      */
int64_t ntco_grid_offset(const ntco_desc* d, int32_t level, int32_t k) {
    int64_t off = 0;
    for (int32_t j = 0; j <= level; ++j) {
        int32_t r0, r1;
        ntco_grid_res(d, j, &r0, &r1);
        for (int32_t kk = 0; kk < 2; ++kk) {
            if (j == level && kk == k) return off;
            off += kk == 0 ? (int64_t)r0 * r0 * d->c0 : (int64_t)r1 * r1 * d->c1;
        }
    }
    return off;
}

int64_t ntco_num_latents(const ntco_desc* d) {
    return ntco_grid_offset(d, ntco_num_levels(d), 0);
}

/* "The size of our input is given by 4C_0 + C_1 + 12 + 1". */
int32_t ntco_input_dim(const ntco_desc* d) { return 4 * d->c0 + d->c1 + 12 + 1; }

int64_t ntco_num_params(const ntco_desc* d) {
    int64_t D = ntco_input_dim(d);
    return HIDDEN * D + HIDDEN + (int64_t)d->hidden_mats * (HIDDEN * HIDDEN + HIDDEN) +
           (int64_t)d->channels * HIDDEN + d->channels;
}

static int32_t clampi(int32_t v, int32_t lo, int32_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* R1/R2/R3: texel-centre mapping u = (x+1/2) r / w_m - 1/2, clamp-to-edge taps in the
 * order (i,j), (i+1,j), (i,j+1), (i+1,j+1); G_0 taps unweighted ("learned interpolation",
 * PAPER.md:450-452), G_1 taps bilinear.                          */
void ntco_address(const ntco_desc* d, int32_t mip, int32_t x, int32_t y,
                  int32_t out_i[17], double out_w[4]) {
    int32_t j = ntco_level_of_mip(d, mip);
    int32_t r[2];
    ntco_grid_res(d, j, &r[0], &r[1]);
    double wm = (double)(d->width >> mip);
    out_i[0] = j;
    for (int32_t k = 0; k < 2; ++k) {
        double u = ((double)x + 0.5) * (double)r[k] / wm - 0.5;
        double v = ((double)y + 0.5) * (double)r[k] / wm - 0.5;
        double fu = floor(u), fv = floor(v);
        int32_t i0 = (int32_t)fu, j0 = (int32_t)fv;
        for (int32_t t = 0; t < 4; ++t) {
            int32_t ti = clampi(i0 + (t & 1), 0, r[k] - 1);
            int32_t tj = clampi(j0 + (t >> 1), 0, r[k] - 1);
            out_i[1 + 8 * k + 2 * t] = ti;
            out_i[2 + 8 * k + 2 * t] = tj;
        }
        if (k == 1) {
            double ax = u - fu, ay = v - fv;
            out_w[0] = (1.0 - ax) * (1.0 - ay);
            out_w[1] = ax * (1.0 - ay);
            out_w[2] = (1.0 - ax) * ay;
            out_w[3] = ax * ay;
        }
    }
}

/* ------------------------------------------------------------------------- */
/* Quantisation                                            */
/* ------------------------------------------------------------------------- */
/* Range [-(N-1)/2 Q, N/2 Q], N = 2^B, Q = 1/N.  Representable
 * values are the bin centres idx*Q, idx in [-(N/2-1), N/2] (zero is a centre).
 * R9: nearest centre, ties upward (lo is always a tie); code = idx + N/2 - 1 (R10). */
double ntco_quant_lo(int32_t bits) { double N = ldexp(1.0, bits); return -(N - 1.0) / 2.0 / N; }
double ntco_quant_hi(int32_t bits) { double N = ldexp(1.0, bits); return N / 2.0 / N; }

int32_t ntco_quantize(double v, int32_t bits) {
    int32_t N = 1 << bits;
    double Q = 1.0 / (double)N;
    double idx = floor(v / Q + 0.5);
    double lo_idx = -(N / 2 - 1), hi_idx = N / 2;
    if (idx < lo_idx) idx = lo_idx;
    if (idx > hi_idx) idx = hi_idx;
    return (int32_t)idx + N / 2 - 1;
}

double ntco_dequantize(int32_t code, int32_t bits) {
    int32_t N = 1 << bits;
    return (double)(code - (N / 2 - 1)) / (double)N;
}

void ntco_quantize_latents(const ntco_desc* d, const float* latents, uint8_t* codes) {
    int32_t L = ntco_num_levels(d);
    for (int32_t j = 0; j < L; ++j)
        for (int32_t k = 0; k < 2; ++k) {
            int64_t a = ntco_grid_offset(d, j, k), b = ntco_grid_offset(d, j + (k == 1), k == 1 ? 0 : 1);
            int32_t bits = k == 0 ? d->b0 : d->b1;
            for (int64_t i = a; i < b; ++i) codes[i] = (uint8_t)ntco_quantize((double)latents[i], bits);
        }
}

/* ------------------------------------------------------------------------- */
/* fp16 conversion (IEEE 754 binary16)                                       */
/* ------------------------------------------------------------------------- */
uint16_t ntco_f64_to_f16(double v) {
    uint16_t sign = signbit(v) ? 0x8000u : 0u;
    if (isnan(v)) return (uint16_t)(sign | 0x7E00u);
    double a = fabs(v);
    if (a == 0.0) return sign;
    if (a >= 65520.0) return (uint16_t)(sign | 0x7C00u); /* rounds to infinity */
    int e2;
    frexp(a, &e2);            /* a in [2^(e2-1), 2^e2) */
    int32_t E = e2 - 1;       /* unbiased exponent of a */
    int32_t sub = E < -14;
    double quantum = sub ? ldexp(1.0, -24) : ldexp(1.0, E - 10);
    double q = a / quantum;   /* exact: power-of-two division */
    double r = floor(q), frac = q - r;
    if (frac > 0.5 || (frac == 0.5 && fmod(r, 2.0) == 1.0)) r += 1.0;
    if (sub) return (uint16_t)(sign | (uint16_t)r);   /* r == 1024 encodes 2^-14 */
    if (r == 2048.0) { r = 1024.0; E += 1; }
    if (E + 15 >= 31) return (uint16_t)(sign | 0x7C00u);
    return (uint16_t)(sign | (uint16_t)((E + 15) << 10) | (uint16_t)(r - 1024.0));
}

double ntco_f16_to_f64(uint16_t h) {
    int32_t s = h >> 15, e = (h >> 10) & 31, m = h & 1023;
    double v;
    if (e == 0) v = ldexp((double)m, -24);
    else if (e == 31) v = m ? NAN : INFINITY;
    else v = ldexp((double)(1024 + m), e - 25);
    return s ? -v : v;
}

/* ------------------------------------------------------------------------- */
/* Positional encoding and LOD                   */
/* ------------------------------------------------------------------------- */
/* R5: triangle wave of period 1 with tri(0) = 1 (the "triangular waves" of Mueller et al.,
 * PAPER.md:461); 3 octaves (log2 8) x 2 phases (0, 1/4) per axis, at integer
 * texel positions inside the 8x8 tile (Fig 5 caption PAPER.md:468).     */
double ntco_tri(double t) {
    double f = t - floor(t);
    return 4.0 * fabs(f - 0.5) - 1.0;
}

void ntco_pe(int32_t x, int32_t y, double out[12]) {
    int32_t p[2] = {((x % 8) + 8) % 8, ((y % 8) + 8) % 8};
    for (int32_t a = 0; a < 2; ++a)
        for (int32_t h = 0; h < 3; ++h) {
            double t = (double)(1 << h) * (double)p[a] / 8.0;
            out[6 * a + 2 * h + 0] = ntco_tri(t);
            out[6 * a + 2 * h + 1] = ntco_tri(t - 0.25);
        }
}

/* R6: normalised LOD = m / (M-1) (0 for a 1-mip chain), as the fp16 network input. */
uint16_t ntco_lod_f16(int32_t mip, int32_t num_mips) {
    double l = num_mips > 1 ? (double)mip / (double)(num_mips - 1) : 0.0;
    return ntco_f64_to_f16(l);
}

/* Fig 3c: [G0 taps (tap-major, channel-minor) | bilinear G1 | PE_x | PE_y | LOD]
 * (R4).  Each value is rounded to fp16, the network input format (R14).            */
static void assemble_from(const ntco_desc* d, int32_t mip, int32_t x, int32_t y,
                          const uint8_t* codes, const float* latents, const double* noise_tab,
                          int32_t round_f16, double* Xd, int32_t taps[17], double w[4]) {
    ntco_address(d, mip, x, y, taps, w);
    int32_t j = taps[0], r0, r1;
    ntco_grid_res(d, j, &r0, &r1);
    int64_t off0 = ntco_grid_offset(d, j, 0), off1 = ntco_grid_offset(d, j, 1);
    int32_t n = 0;
    for (int32_t t = 0; t < 4; ++t)
        for (int32_t ch = 0; ch < d->c0; ++ch) {
            int64_t li = off0 + ((int64_t)taps[2 + 2 * t] * r0 + taps[1 + 2 * t]) * d->c0 + ch;
            double v = codes ? ntco_dequantize(codes[li], d->b0)
                             : (double)latents[li] + (noise_tab ? noise_tab[li] : 0.0);
            Xd[n++] = v;
        }
    for (int32_t ch = 0; ch < d->c1; ++ch) {
        double s = 0.0;
        for (int32_t t = 0; t < 4; ++t) {
            int64_t li = off1 + ((int64_t)taps[10 + 2 * t] * r1 + taps[9 + 2 * t]) * d->c1 + ch;
            double v = codes ? ntco_dequantize(codes[li], d->b1)
                             : (double)latents[li] + (noise_tab ? noise_tab[li] : 0.0);
            s += w[t] * v;
        }
        Xd[n++] = s;
    }
    double pe[12];
    ntco_pe(x, y, pe);
    for (int32_t i = 0; i < 12; ++i) Xd[n++] = pe[i];
    Xd[n++] = ntco_f16_to_f64(ntco_lod_f16(mip, ntco_num_mips(d->width)));
    if (round_f16)
        for (int32_t i = 0; i < n; ++i) Xd[i] = ntco_f16_to_f64(ntco_f64_to_f16(Xd[i]));
}

void ntco_assemble(const ntco_desc* d, const uint8_t* codes, int32_t mip, int32_t x, int32_t y,
                   uint16_t* X) {
    double Xd[128], w[4];
    int32_t taps[17];
    assemble_from(d, mip, x, y, codes, NULL, NULL, 1, Xd, taps, w);
    for (int32_t i = 0; i < ntco_input_dim(d); ++i) X[i] = ntco_f64_to_f16(Xd[i]);
}

/* ------------------------------------------------------------------------- */
/* Network                                                 */
/* ------------------------------------------------------------------------- */
/* hardGELU piecewise definition; +-3/2 belong to the middle case. */
double ntco_hardgelu(double x) {
    if (x < -1.5) return 0.0;
    if (x > 1.5) return x;
    return x / 3.0 * (x + 1.5);
}

/* R15: derivative of the piecewise definition; at the kinks the middle piece's slope. */
double ntco_hardgelu_grad(double x) {
    if (x < -1.5) return 0.0;
    if (x > 1.5) return 1.0;
    return (2.0 * x + 1.5) / 3.0;
}

/* Exact GELU (Hendrycks & Gimpel): x Phi(x) = x/2 (1 + erf(x/sqrt 2));
 * the `activation = 1` variant.                                  */
double ntco_gelu(double x) { return 0.5 * x * (1.0 + erf(x / sqrt(2.0))); }

/* d/dx x Phi(x) = Phi(x) + x phi(x). */
double ntco_gelu_grad(double x) {
    const double Phi = 0.5 * (1.0 + erf(x / sqrt(2.0)));
    const double phi = exp(-0.5 * x * x) / sqrt(2.0 * 3.14159265358979323846);
    return Phi + x * phi;
}

static double act(int32_t a, double x) { return a == 1 ? ntco_gelu(x) : ntco_hardgelu(x); }
static double act_grad(int32_t a, double x) { return a == 1 ? ntco_gelu_grad(x) : ntco_hardgelu_grad(x); }

typedef struct {
    const double *W[4], *b[4];  /* layers: D->64, (64->64) x hidden_mats, 64->c */
    int32_t nin[4], nout[4], nl;
    int32_t act;                /* 0 hardGELU, 1 GELU */
} mlp_view;

static mlp_view mlp_layout(const ntco_desc* d, const double* params) {
    mlp_view v;
    int32_t D = ntco_input_dim(d);
    v.nl = 2 + d->hidden_mats;
    v.act = d->activation;
    const double* p = params;
    for (int32_t l = 0; l < v.nl; ++l) {
        v.nin[l] = l == 0 ? D : HIDDEN;
        v.nout[l] = l == v.nl - 1 ? d->channels : HIDDEN;
        v.W[l] = p; p += (int64_t)v.nin[l] * v.nout[l];
        v.b[l] = p; p += v.nout[l];
    }
    return v;
}

/* Affine layers with hardGELU (or GELU, activation = 1) after every layer but the last ("We do not use any
 * activation function on the output of the last layer").           */
static void mlp_forward_keep(const mlp_view* v, const double* X, double z[4][HIDDEN],
                             double h[4][HIDDEN], double* y) {
    const double* in = X;
    for (int32_t l = 0; l < v->nl; ++l) {
        double* out = l == v->nl - 1 ? y : z[l];
        for (int32_t o = 0; o < v->nout[l]; ++o) {
            double s = v->b[l][o];
            for (int32_t i = 0; i < v->nin[l]; ++i) s += v->W[l][(int64_t)o * v->nin[l] + i] * in[i];
            out[o] = s;
        }
        if (l < v->nl - 1) {
            for (int32_t o = 0; o < HIDDEN; ++o) h[l][o] = act(v->act, z[l][o]);
            in = h[l];
        }
    }
}

void ntco_mlp_forward(const ntco_desc* d, const double* params, const double* X, double* y) {
    mlp_view v = mlp_layout(d, params);
    double z[4][HIDDEN], h[4][HIDDEN];
    mlp_forward_keep(&v, X, z, h, y);
}

static double* params_from_f16(const ntco_desc* d, const uint16_t* w) {
    int64_t P = ntco_num_params(d);
    double* p = (double*)malloc(sizeof(double) * P);
    for (int64_t i = 0; i < P; ++i) p[i] = ntco_f16_to_f64(w[i]);
    return p;
}

/* ------------------------------------------------------------------------- */
/* Decode                                                                     */
/* ------------------------------------------------------------------------- */
static void decode_one(const ntco_desc* d, const uint8_t* codes, const double* params,
                       int32_t x, int32_t y, int32_t mip, double* out) {
    double Xd[128], w[4], yv[16];
    int32_t taps[17];
    assemble_from(d, mip, x, y, codes, NULL, NULL, 1, Xd, taps, w);
    ntco_mlp_forward(d, params, Xd, yv);
    /* R13: decoded channels are stored clamped to [0,1] (texture values). */
    for (int32_t c = 0; c < d->channels; ++c) out[c] = yv[c] < 0.0 ? 0.0 : (yv[c] > 1.0 ? 1.0 : yv[c]);
}

void ntco_decode_texels(const ntco_desc* d, const uint8_t* codes, const uint16_t* weights_f16,
                        const int32_t* q, int64_t n, double* out, int32_t nthreads) {
    double* params = params_from_f16(d, weights_f16);
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t i = 0; i < n; ++i)
        decode_one(d, codes, params, q[3 * i], q[3 * i + 1], q[3 * i + 2], out + i * d->channels);
    free(params);
}

void ntco_decode_mip(const ntco_desc* d, const uint8_t* codes, const uint16_t* weights_f16,
                     int32_t mip, double* out, int32_t nthreads) {
    double* params = params_from_f16(d, weights_f16);
    int32_t wm = d->width >> mip;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t i = 0; i < (int64_t)wm * wm; ++i)
        decode_one(d, codes, params, (int32_t)(i % wm), (int32_t)(i / wm), mip, out + i * d->channels);
    free(params);
}

/* ------------------------------------------------------------------------- */
/* Filtering                                               */
/* ------------------------------------------------------------------------- */
static double jitter_word(uint32_t w) { return ldexp((double)(2 * (w >> 9) + 1), -24) - 0.5; }

/* bilinear filter of mip m at texture coordinate (u, v): texel centres at (i + 1/2)/w_m,
 * clamp-to-edge (the same convention as the latent grids, R1-R2)                    */
static void bilinear_at(const ntco_desc* d, const uint8_t* codes, const double* params, int32_t m, double u,
                        double v, double* out) {
    int32_t wm = d->width >> m;
    double s = u * wm - 0.5, t = v * wm - 0.5;
    double fs = floor(s), ft = floor(t);
    double a = s - fs, b = t - ft;
    int32_t i = (int32_t)fs, j = (int32_t)ft;
    double w[4] = {(1 - a) * (1 - b), a * (1 - b), (1 - a) * b, a * b};
    double y[16];
    for (int32_t c = 0; c < d->channels; ++c) out[c] = 0.0;
    for (int32_t k = 0; k < 4; ++k) {
        int32_t x = clampi(i + (k & 1), 0, wm - 1), yy = clampi(j + (k >> 1), 0, wm - 1);
        decode_one(d, codes, params, x, yy, m, y);
        for (int32_t c = 0; c < d->channels; ++c) out[c] += w[k] * y[c];
    }
}

void ntco_filter(const ntco_desc* d, const uint8_t* codes, const uint16_t* weights_f16, const double* uvl,
                 int64_t n, int32_t mode, uint64_t seed, double* out, int32_t nthreads) {
    double* params = params_from_f16(d, weights_f16);
    int32_t M = ntco_num_mips(d->width);
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t i = 0; i < n; ++i) {
        double u = uvl[3 * i], v = uvl[3 * i + 1], lod = uvl[3 * i + 2];
        double* o = out + i * d->channels;
        uint32_t ctr[4] = {(uint32_t)i, (uint32_t)((uint64_t)i >> 32), 0u, 0x46494C54u /* 'FILT' */};
        uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
        uint32_t r[4];
        ntco_philox4x32_10(ctr, key, r);
        if (mode == 4) lod += jitter_word(r[2]);
        if (mode == 0 || mode == 3 || mode == 4) {
            int32_t m = clampi((int32_t)floor(lod + 0.5), 0, M - 1), wm = d->width >> m;
            double su = u * wm, sv = v * wm;
            if (mode != 0) { su += jitter_word(r[0]); sv += jitter_word(r[1]); }
            decode_one(d, codes, params, clampi((int32_t)floor(su), 0, wm - 1), clampi((int32_t)floor(sv), 0, wm - 1),
                       m, o);
        } else if (mode == 1) {
            bilinear_at(d, codes, params, clampi((int32_t)floor(lod + 0.5), 0, M - 1), u, v, o);
        } else {
            double fl = floor(lod);
            int32_t m0 = clampi((int32_t)fl, 0, M - 1), m1 = clampi(m0 + 1, 0, M - 1);
            double t = (lod >= M - 1) ? 0.0 : (lod < 0 ? 0.0 : lod - fl);
            double y0[16], y1[16];
            bilinear_at(d, codes, params, m0, u, v, y0);
            bilinear_at(d, codes, params, m1, u, v, y1);
            for (int32_t c = 0; c < d->channels; ++c) o[c] = (1 - t) * y0[c] + t * y1[c];
        }
    }
    free(params);
}

/* ------------------------------------------------------------------------- */
/* Training                                                                   */
/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon et al., SC'11), the counter-based generator both sides implement. */
void ntco_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3], k0 = key[0], k1 = key[1];
    for (int32_t r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1, n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* R16: one U(-Q/2, Q/2) draw per latent per step: word (i mod 4) of
 * Philox(key = seed, ctr = (i/4, i/2^34, step, 'NOIS')); u = (2k+1) 2^-24, k = word >> 9. */
double ntco_noise(uint64_t seed, uint32_t step, int64_t idx, int32_t bits) {
    uint32_t ctr[4] = {(uint32_t)((uint64_t)idx >> 2), (uint32_t)((uint64_t)idx >> 34), step, 0x4E4F4953u};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    ntco_philox4x32_10(ctr, key, o);
    double u = ldexp((double)(2 * (o[idx & 3] >> 9) + 1), -24);
    return (u - 0.5) / (double)(1 << bits);
}

static int32_t is_g1_index(const ntco_desc* d, int64_t li, int32_t* bits) {
    int32_t L = ntco_num_levels(d);
    for (int32_t j = 0; j < L; ++j) {
        if (li < ntco_grid_offset(d, j, 1)) { *bits = d->b0; return 0; }
        if (li < ntco_grid_offset(d, j + 1, 0)) { *bits = d->b1; return 1; }
    }
    *bits = d->b1;
    return 1;
}

/* One batch: crops at one LOD, noisy latents, MLP with the
 * weights in the fp16 format the tensor cores consume (R14), mean L2 loss
 * (R17), analytic backward through the MLP, concatenation, bilinear weights
 * and additive noise.                                            */
double ntco_train_grads(const ntco_desc* d, const float* latents, const float* params_f32,
                        int32_t mip, int32_t n_crops, const int32_t* crops,
                        const uint16_t* ref_f16, uint64_t seed, uint32_t step, int32_t noise_on,
                        int32_t round_f16, double* dparams, double* dlatents, int32_t nthreads) {
    int64_t P = ntco_num_params(d), NL = ntco_num_latents(d);
    int32_t D = ntco_input_dim(d), c = d->channels, wm = d->width >> mip;
    int32_t nlat_in = 4 * d->c0 + d->c1;
    double* params = (double*)malloc(sizeof(double) * P);
    for (int64_t i = 0; i < P; ++i)
        params[i] = round_f16 ? ntco_f16_to_f64(ntco_f64_to_f16((double)params_f32[i])) : (double)params_f32[i];
    mlp_view v = mlp_layout(d, params);

    /* noise table: one draw per latent per step, shared by every texel reading it */
    double* noise = NULL;
    if (noise_on) {
        noise = (double*)malloc(sizeof(double) * NL);
        for (int64_t i = 0; i < NL; ++i) {
            int32_t bits;
            is_g1_index(d, i, &bits);
            noise[i] = ntco_noise(seed, step, i, bits);
        }
    }

    int64_t B = 0;
    for (int32_t k = 0; k < n_crops; ++k) B += (int64_t)crops[4 * k + 2] * crops[4 * k + 3];
    int64_t* start = (int64_t*)malloc(sizeof(int64_t) * (n_crops + 1));
    start[0] = 0;
    for (int32_t k = 0; k < n_crops; ++k) start[k + 1] = start[k] + (int64_t)crops[4 * k + 2] * crops[4 * k + 3];

    double* dX = (double*)malloc(sizeof(double) * B * nlat_in);
    int32_t* taps = (int32_t*)malloc(sizeof(int32_t) * B * 17);
    double* tw = (double*)malloc(sizeof(double) * B * 4);
    double* sq = (double*)malloc(sizeof(double) * B);
    int32_t nt = 1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
    nt = omp_get_max_threads();
#endif
    double* dpart = (double*)calloc((size_t)nt * P, sizeof(double));
    double inv = 2.0 / ((double)B * (double)c);

#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
    for (int64_t t = 0; t < B; ++t) {
        int32_t tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        double* dp = dpart + (int64_t)tid * P;
        int32_t k = 0;
        while (t >= start[k + 1]) ++k;
        int64_t r = t - start[k];
        int32_t cw = crops[4 * k + 2];
        int32_t x = crops[4 * k] + (int32_t)(r % cw), y = crops[4 * k + 1] + (int32_t)(r / cw);
        double Xd[128], z[4][HIDDEN], h[4][HIDDEN], yv[16];
        assemble_from(d, mip, x, y, NULL, latents, noise, round_f16, Xd, taps + 17 * t, tw + 4 * t);
        mlp_forward_keep(&v, Xd, z, h, yv);
        /* backward; parameter gradient layout mirrors the ABI parameter order */
        double dz[HIDDEN], dh[128];
        double s2 = 0.0;
        for (int32_t o = 0; o < c; ++o) {
            double e = yv[o] - ntco_f16_to_f64(ref_f16[((int64_t)y * wm + x) * c + o]);
            s2 += e * e;
            dz[o] = inv * e;
        }
        sq[t] = s2;
        int64_t poff[4];
        {
            int64_t o = 0;
            for (int32_t l = 0; l < v.nl; ++l) { poff[l] = o; o += (int64_t)v.nin[l] * v.nout[l] + v.nout[l]; }
        }
        for (int32_t l = v.nl - 1; l >= 0; --l) {
            const double* in = l == 0 ? Xd : h[l - 1];
            double* gW = dp + poff[l];
            double* gb = gW + (int64_t)v.nin[l] * v.nout[l];
            for (int32_t o = 0; o < v.nout[l]; ++o) {
                gb[o] += dz[o];
                for (int32_t i = 0; i < v.nin[l]; ++i) gW[(int64_t)o * v.nin[l] + i] += dz[o] * in[i];
            }
            for (int32_t i = 0; i < v.nin[l]; ++i) {
                double s = 0.0;
                for (int32_t o = 0; o < v.nout[l]; ++o) s += v.W[l][(int64_t)o * v.nin[l] + i] * dz[o];
                dh[i] = s;
            }
            if (l > 0)
                for (int32_t i = 0; i < HIDDEN; ++i) dz[i] = dh[i] * act_grad(v.act, z[l - 1][i]);
        }
        for (int32_t i = 0; i < nlat_in; ++i) dX[t * nlat_in + i] = dh[i];
        (void)D;
    }

    /* fixed-order reductions */
    for (int64_t i = 0; i < P; ++i) {
        double s = 0.0;
        for (int32_t q = 0; q < nt; ++q) s += dpart[(int64_t)q * P + i];
        dparams[i] = s;
    }
    memset(dlatents, 0, sizeof(double) * NL);
    double loss = 0.0;
    for (int64_t t = 0; t < B; ++t) {
        loss += sq[t];
        const int32_t* tp = taps + 17 * t;
        int32_t j = tp[0], r0, r1;
        ntco_grid_res(d, j, &r0, &r1);
        int64_t off0 = ntco_grid_offset(d, j, 0), off1 = ntco_grid_offset(d, j, 1);
        /* G_0 taps receive unweighted gradients; G_1 taps bilinear-weighted (R16) */
        for (int32_t q = 0; q < 4; ++q)
            for (int32_t ch = 0; ch < d->c0; ++ch)
                dlatents[off0 + ((int64_t)tp[2 + 2 * q] * r0 + tp[1 + 2 * q]) * d->c0 + ch] +=
                    dX[t * nlat_in + q * d->c0 + ch];
        for (int32_t q = 0; q < 4; ++q)
            for (int32_t ch = 0; ch < d->c1; ++ch)
                dlatents[off1 + ((int64_t)tp[10 + 2 * q] * r1 + tp[9 + 2 * q]) * d->c1 + ch] +=
                    tw[4 * t + q] * dX[t * nlat_in + 4 * d->c0 + ch];
    }
    loss /= (double)B * (double)c;
    free(params); free(noise); free(start); free(dX); free(taps); free(tw); free(sq); free(dpart);
    return loss;
}

/* Adam (Kingma & Ba) with bias correction; R18: beta1=0.9, beta2=0.999,
 * eps=1e-8 by default, sparse mode skips entries whose gradient is exactly zero; the
 * latent clamp to the quantisation range follows the update.       */
void ntco_adam(int64_t n, float* p, float* m, float* v, const float* g, int32_t t,
               double lr, double beta1, double beta2, double eps, int32_t sparse,
               int32_t clamp_on, double lo, double hi) {
    double c1 = 1.0 - pow(beta1, (double)t), c2 = 1.0 - pow(beta2, (double)t);
    for (int64_t i = 0; i < n; ++i) {
        double gi = (double)g[i];
        if (sparse && gi == 0.0) continue;
        double mi = beta1 * (double)m[i] + (1.0 - beta1) * gi;
        double vi = beta2 * (double)v[i] + (1.0 - beta2) * gi * gi;
        double pi = (double)p[i] - lr * (mi / c1) / (sqrt(vi / c2) + eps);
        if (clamp_on) pi = pi < lo ? lo : (pi > hi ? hi : pi);
        m[i] = (float)mi;
        v[i] = (float)vi;
        p[i] = (float)pi;
    }
}
