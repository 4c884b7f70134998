/*
 * turbo_oracle.c -- plain, slow, scalar CPU oracle for TurboAttention
 * (arXiv 2412.08585).  TEST INFRASTRUCTURE ONLY (see turbo_oracle.h).
 *
 * Built with -O2 -ffp-contract=off and no fast-math so that every float
 * expression below is evaluated exactly as written (IEEE binary32, round to
 * nearest even), with fused multiply-adds only where fmaf() is written.
 *
 * Precision: the paper fixes the stage-1 codes to INT8 with divisor 119
 * (Alg. 1), stage-2 to INT4/INT2 integers, and runs the
 * score/softmax arithmetic in a GPU float format.  Readings
 * R-1..R-28 pin the float arithmetic to binary32; the running
 * output O and row sum l are kept in double here (they are in the tolerance
 * set, not the exact set).
 */
#include "turbo_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define TQ_DIV 119.0f /* Alg. 1: s = max(abs(X)) / 119 */

/* IEEE binary16 rounding (nearest, ties to even) of a float, returned as a float: the
 * first-stage scales of the scale_fp16 variant ("FP16" scales; R-29).  Written out
 * from the format's definition: 11 significant bits, quantum 2^(e-11) for |s| in
 * [2^(e-1), 2^e), never finer than the subnormal quantum 2^-24, overflow past 65504. */
static float round_fp16(float s) {
  double a = fabs((double)s);
  if (a == 0.0 || !isfinite(a)) return s;
  int e;
  frexp(a, &e);
  int q = e - 11;
  if (q < -24) q = -24;
  double r = ldexp(rint(ldexp(a, -q)), q);  /* rint: round half to even (default mode) */
  if (r > 65504.0) r = INFINITY;
  return (float)(s < 0.0f ? -r : r);
}

/* binary16 fused multiply-add: the binary16 rounding (nearest even) of the EXACT a*b + c
 * for binary16 values a, b, c (sas_fp16 variant, R-30).  Every binary16 value is an integer
 * multiple of 2^-24, so a*b + c = K 2^-48 with |K| < 2^81: K is formed exactly in 128-bit
 * integers and rounded once, with the quantum rule of round_fp16. */
static float fma_fp16(float a, float b, float c) {
  const __int128 ka = (__int128)ldexp((double)a, 24), kb = (__int128)ldexp((double)b, 24);
  const __int128 kc = (__int128)ldexp((double)c, 24);
  const __int128 K = ka * kb + kc * ((__int128)1 << 24);
  if (K == 0) return 0.0f;
  unsigned __int128 m = (unsigned __int128)(K < 0 ? -K : K);
  int e = 0;                                   /* |K| in [2^(e-1), 2^e) */
  while (e < 127 && (m >> e) != 0) ++e;
  int q = (e - 48) - 11;                       /* quantum exponent of the result */
  if (q < -24) q = -24;
  const int sh = q + 48;                       /* >= 24: drop sh bits of K */
  unsigned __int128 r = m >> sh;
  const unsigned __int128 rem = m & (((unsigned __int128)1 << sh) - 1), half = (unsigned __int128)1 << (sh - 1);
  if (rem > half || (rem == half && (r & 1))) ++r;
  double v = ldexp((double)(uint64_t)r, q);
  if (v > 65504.0) v = INFINITY;
  return (float)(K < 0 ? -v : v);
}

/* ------------------------------------------------------------------------ */
/* SAS: e^{-x} ~= LUT(x_int) * POLY(x_dec), 0 below the threshold n_r.       */
/* ------------------------------------------------------------------------ */

/* LUT[i] = e^{-i}, i = 0..|n_r|, correctly rounded to binary32 (P:462-466,
 * Appendix B "look-up table T"). */
void tq_sas_lut(int32_t nr, float* lut) {
  for (int32_t i = 0; i <= -nr; ++i) lut[i] = (float)exp(-(double)i);
}

/* POLY(x) = -0.1025 x^3 + 0.4626 x^2 - 0.9922 x + 0.9996 on [0,1],
 * evaluated by Horner with one rounding per step (R-13). */
float tq_sas_poly(float f) {
  const float c3 = -0.1025f, c2 = 0.4626f, c1 = -0.9922f, c0 = 0.9996f;
  return fmaf(fmaf(fmaf(c3, f, c2), f, c1), f, c0);
}

/* SAS applied to dist = m - x >= 0, i.e. SAS(x - m) of P:468-470:
 *   0                         if x - m < n_r     (dist > -n_r, strict; R-12)
 *   LUT[int] * POLY(dec)      otherwise, int = floor(dist), dec = dist - int. */
float tq_sas(float dist, int32_t nr) {
  if (dist > (float)(-nr)) return 0.0f;
  float fi = floorf(dist);
  int32_t i = (int32_t)fi;
  float f = dist - fi;                     /* exact (Sterbenz / fi == 0) */
  float lut_i = (float)exp(-(double)i);    /* = LUT[i] of tq_sas_lut */
  return lut_i * tq_sas_poly(f);
}

/* sas_fp16 variant (the polynomial "in FP16"; R-30): the same threshold, floor and
 * exact fraction, then f and the four printed coefficients rounded to binary16 and POLY by
 * Horner with binary16 fused multiply-adds; the LUT factor and the product stay binary32. */
float tq_sas_poly_fp16(float f) {
  const float c3 = round_fp16(-0.1025f), c2 = round_fp16(0.4626f), c1 = round_fp16(-0.9922f),
              c0 = round_fp16(0.9996f);
  const float fh = round_fp16(f);
  return fma_fp16(fma_fp16(fma_fp16(c3, fh, c2), fh, c1), fh, c0);
}

float tq_sas_fp16(float dist, int32_t nr) {
  if (dist > (float)(-nr)) return 0.0f;
  float fi = floorf(dist);
  int32_t i = (int32_t)fi;
  float f = dist - fi;
  float lut_i = (float)exp(-(double)i);
  return lut_i * tq_sas_poly_fp16(f);
}

/* The SAS a parameter set selects (FP32 Horner, or the sas_fp16 variant). */
static float sas_p(const tq_params* p, float dist) {
  return p->sas_fp16 ? tq_sas_fp16(dist, p->sas_nr) : tq_sas(dist, p->sas_nr);
}

/* Appendix B: row-normalised SAS softmax.  Step 1 subtract the
 * row max, step 2 threshold, steps 3-4 LUT x POLY, step 5 divide by row sum. */
void tq_sas_softmax_rows(int32_t rows, int32_t cols, const float* x, int32_t nr, float* out) {
  for (int32_t r = 0; r < rows; ++r) {
    const float* xr = x + (int64_t)r * cols;
    float* orow = out + (int64_t)r * cols;
    float mx = -INFINITY;
    for (int32_t c = 0; c < cols; ++c) mx = fmaxf(mx, xr[c]);
    double sum = 0.0;
    for (int32_t c = 0; c < cols; ++c) {
      orow[c] = tq_sas(mx - xr[c], nr);
      sum += orow[c];
    }
    for (int32_t c = 0; c < cols; ++c) orow[c] = (float)(orow[c] / sum);
  }
}


/* A first-stage scale as used and stored: FP32, or its FP16 rounding (scale_fp16). */
static float st1(const tq_params* p, float s) { return p->scale_fp16 ? round_fp16(s) : s; }

/* ------------------------------------------------------------------------ */
/* FlashQ stage 1: symmetric INT8 per block (Eq. 9; Alg. 1) */
/* ------------------------------------------------------------------------ */

/* s = max|x| / 119;  code = round_half_even(x * (119 / max|x|)) with the
 * product taken exactly (R-2, R-3).  All-zero block: s = 0, codes 0 (R-5). */
void tq_quant_sym8(const float* x, int64_t n, int8_t* codes, float* s_out) {
  float a = 0.0f;
  for (int64_t i = 0; i < n; ++i) a = fmaxf(a, fabsf(x[i]));
  if (a == 0.0f) {
    for (int64_t i = 0; i < n; ++i) codes[i] = 0;
    *s_out = 0.0f;
    return;
  }
  float inv = TQ_DIV / a;
  *s_out = a / TQ_DIV;
  for (int64_t i = 0; i < n; ++i) codes[i] = (int8_t)rint((double)x[i] * (double)inv);
}

/* ------------------------------------------------------------------------ */
/* FlashQ stage 2: asymmetric INT4/INT2, integer only (Eq. 10;     */
/* Alg. 1; Eq. 7-8; R-6)                                  */
/* ------------------------------------------------------------------------ */

/* One group = one channel of one B_c block (R-7).  z = min, s = max(1,
 * ceil((max-min)/(2^b-1))), code = round_half_up((g - z)/s). */
void tq_quant_asym(const int8_t* g, int32_t n, int64_t stride, int32_t bits, uint8_t* codes,
                   int64_t code_stride, uint8_t* s_int, int8_t* z_int) {
  int32_t mn = 127, mx = -128;
  for (int32_t t = 0; t < n; ++t) {
    int32_t v = g[(int64_t)t * stride];
    if (v < mn) mn = v;
    if (v > mx) mx = v;
  }
  int32_t levels = (1 << bits) - 1;
  int32_t s = (mx - mn + levels - 1) / levels;
  if (s < 1) s = 1;
  for (int32_t t = 0; t < n; ++t) {
    int32_t v = g[(int64_t)t * stride];
    codes[(int64_t)t * code_stride] = (uint8_t)((2 * (v - mn) + s) / (2 * s));
  }
  *s_int = (uint8_t)s;
  *z_int = (int8_t)mn;
}

/* Integer dequantisation back to INT8: K^q1 = K^q2 * s^int + z^int (Alg. 2
 * P:966-967, Eq. 7-8). */
int32_t tq_dequant_q2(int32_t code, int32_t s_int, int32_t z_int) { return code * s_int + z_int; }

/* ------------------------------------------------------------------------ */
/* KV cache: prefill construction and decode-time append (Sec. 3.3)          */
/* ------------------------------------------------------------------------ */

static int8_t quant_univ(float x, float a_univ) {
  /* Buffer token: INT8 with the universal scale, outliers clamped. */
  if (a_univ == 0.0f) return 0;
  float inv = TQ_DIV / a_univ;
  double c = rint((double)x * (double)inv);
  if (c > 119.0) c = 119.0;
  if (c < -119.0) c = -119.0;
  return (int8_t)c;
}

static void flush_block(const tq_params* p, tq_slot* s, const int8_t* x1 /*[B_c][d]*/, float parent) {
  int32_t d = p->d, bc = p->block_kv, b = s->n_blocks;
  uint8_t* codes = s->codes + (int64_t)b * bc * d;
  for (int32_t c = 0; c < d; ++c)
    tq_quant_asym(x1 + c, bc, d, s->bits, codes + c, d, s->s_int + (int64_t)b * d + c,
                  s->z_int + (int64_t)b * d + c);
  s->s_parent[b] = parent;
  s->n_blocks = b + 1;
}

/* PREFILL: every B_c block -> stage-1 (x1, x1_scale: the prefill operands);
 * every full block -> stage-2 into the cache with its stage-1 scale as parent
 * (Alg. 1).  The universal scale is the max-abs over the prefill
 * tokens (R-9); the N mod B_c tail goes to the INT8 buffer (R-11). */
int32_t tq_cache_prefill_slot(const tq_params* p, int32_t n, const float* x, tq_slot* s,
                              int8_t* x1, float* x1_scale) {
  int32_t d = p->d, bc = p->block_kv;
  if (n < 1) return -1;
  int32_t tc = (n + bc - 1) / bc, nfull = n / bc;
  if (nfull > s->max_blocks) return -3;
  int8_t* blk = (int8_t*)malloc((size_t)bc * d);
  s->n_blocks = 0;
  float a_univ = 0.0f;
  for (int64_t i = 0; i < (int64_t)n * d; ++i) a_univ = fmaxf(a_univ, fabsf(x[i]));
  s->a_univ = a_univ;
  for (int32_t j = 0; j < tc; ++j) {
    int32_t rows = (j + 1) * bc <= n ? bc : n - j * bc;
    float sc;
    tq_quant_sym8(x + (int64_t)j * bc * d, (int64_t)rows * d, blk, &sc);
    sc = st1(p, sc);
    if (x1) memcpy(x1 + (int64_t)j * bc * d, blk, (size_t)rows * d);
    if (x1_scale) x1_scale[j] = sc;
    if (rows == bc) flush_block(p, s, blk, sc);
  }
  s->n_buf = n - nfull * bc;
  for (int32_t t = 0; t < s->n_buf; ++t)
    for (int32_t c = 0; c < d; ++c)
      s->buf[(int64_t)t * d + c] = quant_univ(x[((int64_t)nfull * bc + t) * d + c], a_univ);
  free(blk);
  return 0;
}

/* PREFILL of a further chunk (R-28): the slot must hold whole blocks only
 * (n_buf = 0).  The universal scale becomes the max-abs over every prefill
 * chunk so far (R-9); the chunk's blocks are stage-1 quantised (the chunked
 * prefill's operands) and its full blocks appended after the existing ones;
 * its tail goes to the INT8 buffer with the updated universal scale. */
int32_t tq_cache_prefill_append_slot(const tq_params* p, int32_t n, const float* x, tq_slot* s,
                                     int8_t* x1, float* x1_scale) {
  int32_t d = p->d, bc = p->block_kv;
  if (n < 1) return -1;
  if (s->n_buf != 0) {
    /* R-31: a chunk that starts inside a block first completes that block exactly as decode
     * appends do (universal scale, clamp +-119, flushed at B_c with parent s_univ);
     * those tokens' stage-1 operands are their buffer codes, at the boundary block's scale
     * s_univ (listed with the prefix, stage1_prefix); the rest of the chunk is block-aligned. */
    int32_t r = bc - s->n_buf < n ? bc - s->n_buf : n;
    for (int32_t t = 0; t < r; ++t) {
      if (x1)
        for (int32_t c = 0; c < d; ++c) x1[(int64_t)t * d + c] = quant_univ(x[(int64_t)t * d + c], s->a_univ);
      int32_t rc = tq_cache_append_slot(p, x + (int64_t)t * d, s);
      if (rc != 0) return rc;
    }
    if (r == n) return 0;
    return tq_cache_prefill_append_slot(p, n - r, x + (int64_t)r * d, s, x1 ? x1 + (int64_t)r * d : x1, x1_scale);
  }
  int32_t tc = (n + bc - 1) / bc, nfull = n / bc;
  if (s->n_blocks + nfull > s->max_blocks) return -3;
  int8_t* blk = (int8_t*)malloc((size_t)bc * d);
  float a_univ = s->a_univ;
  for (int64_t i = 0; i < (int64_t)n * d; ++i) a_univ = fmaxf(a_univ, fabsf(x[i]));
  s->a_univ = a_univ;
  for (int32_t j = 0; j < tc; ++j) {
    int32_t rows = (j + 1) * bc <= n ? bc : n - j * bc;
    float sc;
    tq_quant_sym8(x + (int64_t)j * bc * d, (int64_t)rows * d, blk, &sc);
    sc = st1(p, sc);
    if (x1) memcpy(x1 + (int64_t)j * bc * d, blk, (size_t)rows * d);
    if (x1_scale) x1_scale[j] = sc;
    if (rows == bc) flush_block(p, s, blk, sc);
  }
  s->n_buf = n - nfull * bc;
  for (int32_t t = 0; t < s->n_buf; ++t)
    for (int32_t c = 0; c < d; ++c)
      s->buf[(int64_t)t * d + c] = quant_univ(x[((int64_t)nfull * bc + t) * d + c], a_univ);
  free(blk);
  return 0;
}

/* The universal scale s_univ = a_univ / 119 as used (the buffer block's and a flushed buffer's
 * scale; FP16 variant: R-29). */
float tq_slot_univ_scale(const tq_params* p, const tq_slot* s) { return st1(p, s->a_univ / TQ_DIV); }

/* APPEND one decode token (append, then attend).  When the buffer
 * reaches n_b = B_c tokens it is progressively quantised with the universal
 * scale as its parent scale. */
int32_t tq_cache_append_slot(const tq_params* p, const float* x, tq_slot* s) {
  int32_t d = p->d, bc = p->block_kv;
  if (s->n_buf == bc - 1 && s->n_blocks >= s->max_blocks) return -3;
  for (int32_t c = 0; c < d; ++c) s->buf[(int64_t)s->n_buf * d + c] = quant_univ(x[c], s->a_univ);
  s->n_buf += 1;
  if (s->n_buf == bc) {
    flush_block(p, s, s->buf, st1(p, s->a_univ / TQ_DIV));
    s->n_buf = 0;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Online-softmax tile step shared by prefill and decode (Alg. 1,  */
/* Alg. 2).                                                        */
/* ------------------------------------------------------------------------ */

static float expo(const tq_params* p, float dist) {
  /* P~ = SAS(x - m), or the exact exponential under the P5 switch. */
  return p->sas ? sas_p(p, dist) : (float)exp(-(double)dist);
}

/* One row of one tile.  x[c] = -inf marks masked keys.  Returns 0 when the row
 * has no visible key in this tile (then nothing changes, R-20). */
static int32_t row_step(const tq_params* p, int32_t nc, const float* x, float* m, double* l,
                        float* pt, double* alpha_out) {
  float mt = -INFINITY;
  for (int32_t c = 0; c < nc; ++c) mt = fmaxf(mt, x[c]);
  if (mt == -INFINITY) return 0;
  float m_prev = *m;
  float m_new = fmaxf(m_prev, mt);
  double alpha;
  if (m_prev == -INFINITY) alpha = 0.0;
  else if (!p->sas) alpha = exp((double)m_prev - (double)m_new);
  else if (p->alpha_mode == 1 && m_new == m_prev) alpha = 1.0;
  else alpha = (double)sas_p(p, m_new - m_prev);
  double rowsum = 0.0;
  for (int32_t c = 0; c < nc; ++c) {
    pt[c] = x[c] == -INFINITY ? 0.0f : expo(p, m_new - x[c]);
    rowsum += pt[c];
  }
  *l = alpha * (*l) + rowsum;
  *m = m_new;
  *alpha_out = alpha;
  return 1;
}

/* P quantisation (Alg. 1): s_P = max P~ / 119 over the tile,
 * code = round_half_even(P~ * (119 / max P~)) with the product taken exactly. */
static float quant_p(int64_t n, const float* pt, const uint8_t* use, int32_t width, uint8_t* pc) {
  float a = 0.0f;
  for (int64_t i = 0; i < n; ++i)
    if (use[i / width]) a = fmaxf(a, pt[i]);
  if (a == 0.0f) {
    for (int64_t i = 0; i < n; ++i) pc[i] = 0;
    return 0.0f;
  }
  float inv = TQ_DIV / a;
  for (int64_t i = 0; i < n; ++i) pc[i] = use[i / width] ? (uint8_t)rint((double)pt[i] * (double)inv) : 0;
  return a / TQ_DIV;
}

/* ------------------------------------------------------------------------ */
/* Algorithm 1: TurboAttention prefill, one (batch, head)         */
/* ------------------------------------------------------------------------ */

int32_t tq_prefill_head(const tq_params* p, int32_t n, int32_t causal, const float* q,
                        const float* k, const float* v, float* o, float* lse,
                        tq_prefill_tap* tap) {
  return tq_prefill_head_blocks(p, n, causal, q, k, v, 0, INT32_MAX, o, lse, tap);
}

/* Alg. 1's outer loop restricted to query blocks i in [i_begin, i_end): every
 * iteration of that loop is independent, so this computes exactly
 * the same rows as the full call; rows of other blocks are left untouched. */
/* Alg. 1 for nq query rows at absolute positions q0 .. q0+nq-1
 * against nk keys given as stage-1 operands k1, v1 (int8 [nk][d]) with block
 * scales sk, sv [ceil(nk / B_c)]; k, v (raw [nk][d]) are read only in exact
 * mode (quant = 0).  The prefill (q0 = 0, nq = nk) and the chunked prefill
 * (R-28) both run this loop. */
static int32_t prefill_core(const tq_params* p, int32_t nq, int32_t nk, int32_t q0, int32_t causal,
                            const float* q, const float* k, const float* v, const int8_t* k1,
                            const int8_t* v1, const float* sk, const float* sv, int32_t i_begin,
                            int32_t i_end, float* o, float* lse, tq_prefill_tap* tap);

int32_t tq_prefill_head_blocks(const tq_params* p, int32_t n, int32_t causal, const float* q,
                               const float* k, const float* v, int32_t i_begin, int32_t i_end,
                               float* o, float* lse, tq_prefill_tap* tap) {
  const int32_t d = p->d, bc = p->block_kv;
  if (n < 1 || i_begin < 0) return -1;
  const int32_t tc = (n + bc - 1) / bc;

  /* Stage-1 K_j, V_j; done once per block instead of once per
   * (i, j) -- identical values (R-21). */
  int8_t* k1 = (int8_t*)malloc((size_t)n * d);
  int8_t* v1 = (int8_t*)malloc((size_t)n * d);
  float* sk = (float*)malloc(sizeof(float) * tc);
  float* sv = (float*)malloc(sizeof(float) * tc);
  for (int32_t j = 0; j < tc; ++j) {
    int32_t rows = (j + 1) * bc <= n ? bc : n - j * bc;
    tq_quant_sym8(k + (int64_t)j * bc * d, (int64_t)rows * d, k1 + (int64_t)j * bc * d, &sk[j]);
    tq_quant_sym8(v + (int64_t)j * bc * d, (int64_t)rows * d, v1 + (int64_t)j * bc * d, &sv[j]);
    sk[j] = st1(p, sk[j]);
    sv[j] = st1(p, sv[j]);
  }
  const int32_t rc = prefill_core(p, n, n, 0, causal, q, k, v, k1, v1, sk, sv, i_begin, i_end, o, lse, tap);
  free(k1); free(v1); free(sk); free(sv);
  return rc;
}

int32_t tq_prefill_chunk_head(const tq_params* p, int32_t nq, int32_t nk, int32_t causal, const float* q,
                              const int8_t* k1, const float* sk, const int8_t* v1, const float* sv,
                              float* o, float* lse) {
  if (nq < 1 || nk < nq || !p->quant) return -1;
  return prefill_core(p, nq, nk, nk - nq, causal, q, NULL, NULL, k1, v1, sk, sv, 0, INT32_MAX, o, lse, NULL);
}

static int32_t prefill_core(const tq_params* p, int32_t nq, int32_t nk, int32_t q0, int32_t causal,
                            const float* q, const float* k, const float* v, const int8_t* k1,
                            const int8_t* v1, const float* sk, const float* sv, int32_t i_begin,
                            int32_t i_end, float* o, float* lse, tq_prefill_tap* tap) {
  const int32_t d = p->d, br = p->block_q, bc = p->block_kv;
  const int32_t n = nq;  /* query rows */
  const int32_t tr = (n + br - 1) / br, tc = (nk + bc - 1) / bc;
  if (i_end > tr) i_end = tr;

  int8_t* q1 = (int8_t*)malloc((size_t)br * d);
  float* x = (float*)malloc(sizeof(float) * br * bc);
  int32_t* sint = (int32_t*)malloc(sizeof(int32_t) * br * bc);
  float* pt = (float*)malloc(sizeof(float) * br * bc);
  uint8_t* pc = (uint8_t*)malloc((size_t)br * bc);
  int32_t* pv = (int32_t*)malloc(sizeof(int32_t) * br * d);
  double* O = (double*)malloc(sizeof(double) * br * d);
  double* l = (double*)malloc(sizeof(double) * br);
  double* alpha = (double*)malloc(sizeof(double) * br);
  float* m = (float*)malloc(sizeof(float) * br);
  uint8_t* active = (uint8_t*)malloc((size_t)br);
  float* sp_row = (float*)malloc(sizeof(float) * br);

  for (int32_t i = i_begin; i < i_end; ++i) {    /* for 1 <= i <= T_r */
    const int32_t r0 = i * br, nr = (r0 + br <= n) ? br : n - r0;
    float sq = 0.0f;
    if (p->quant) tq_quant_sym8(q + (int64_t)r0 * d, (int64_t)nr * d, q1, &sq);
    sq = st1(p, sq);
    for (int32_t r = 0; r < nr; ++r) {            /* init O, l, m */
      m[r] = -INFINITY;
      l[r] = 0.0;
      for (int32_t c = 0; c < d; ++c) O[(int64_t)r * d + c] = 0.0;
    }
    const int32_t jmax = causal ? (q0 + r0 + nr - 1) / bc : tc - 1; /* R-20 */
    for (int32_t j = 0; j <= jmax; ++j) {         /* for 1 <= j <= T_c */
      const int32_t c0 = j * bc, nc = (c0 + bc <= nk) ? bc : nk - c0;
      const int32_t tapped = tap && tap->i_block == i && tap->j_block == j;
      /* S = s_Q s_K Q^q1 K^q1^T, scaled by 1/sqrt(d) (R-18). */
      const float cqk = (sq * sk[j]) * p->softmax_scale;
      for (int32_t r = 0; r < nr; ++r)
        for (int32_t c = 0; c < nc; ++c) {
          float* xe = &x[(int64_t)r * bc + c];
          sint[(int64_t)r * bc + c] = 0;
          if (causal && c0 + c > q0 + r0 + r) { *xe = -INFINITY; continue; }
          if (p->quant) {
            int32_t acc = 0;
            for (int32_t e = 0; e < d; ++e)
              acc += (int32_t)q1[(int64_t)r * d + e] * (int32_t)k1[(int64_t)(c0 + c) * d + e];
            sint[(int64_t)r * bc + c] = acc;
            *xe = (float)acc * cqk;
          } else {
            double acc = 0.0;
            for (int32_t e = 0; e < d; ++e)
              acc += (double)q[(int64_t)(r0 + r) * d + e] * (double)k[(int64_t)(c0 + c) * d + e];
            *xe = (float)(acc * (double)p->softmax_scale);
          }
        }
      /* m, P~, l. */
      for (int32_t r = 0; r < nr; ++r)
        active[r] = (uint8_t)row_step(p, nc, x + (int64_t)r * bc, &m[r], &l[r],
                                      pt + (int64_t)r * bc, &alpha[r]);
      /* P quantisation over the B_r x B_c tile and O update
       * O = alpha O + s_P s_V Q(P~) V^q1 (R-15, R-16). */
      float sp = 0.0f;
      if (p->quant) {
        for (int32_t r = 0; r < nr; ++r)        /* compact the tile to width nc */
          for (int32_t c = 0; c < nc; ++c) pt[(int64_t)r * nc + c] = pt[(int64_t)r * bc + c];
        if (p->p_row) {                         /* per row x B_c block (P:976-977 granularity) */
          for (int32_t r = 0; r < nr; ++r)
            sp_row[r] = quant_p(nc, pt + (int64_t)r * nc, active + r, nc, pc + (int64_t)r * nc);
          sp = sp_row[0];
        } else {                                /* per B_r x B_c tile */
          sp = quant_p((int64_t)nr * nc, pt, active, nc, pc);
          for (int32_t r = 0; r < nr; ++r) sp_row[r] = sp;
        }
        for (int32_t r = 0; r < nr; ++r)
          for (int32_t e = 0; e < d; ++e) {
            int32_t acc = 0;
            for (int32_t c = 0; c < nc; ++c)
              acc += (int32_t)pc[(int64_t)r * nc + c] * (int32_t)v1[(int64_t)(c0 + c) * d + e];
            pv[(int64_t)r * d + e] = acc;
          }
        for (int32_t r = 0; r < nr; ++r) {
          if (!active[r]) continue;
          const float cpv = sp_row[r] * sv[j];
          for (int32_t e = 0; e < d; ++e) {
            double* oe = &O[(int64_t)r * d + e];
            *oe = alpha[r] * (*oe) + (double)(cpv * (float)pv[(int64_t)r * d + e]);
          }
        }
      } else {
        for (int32_t r = 0; r < nr; ++r) {
          if (!active[r]) continue;
          for (int32_t e = 0; e < d; ++e) {
            double acc = 0.0;
            for (int32_t c = 0; c < nc; ++c)
              acc += (double)pt[(int64_t)r * bc + c] * (double)v[(int64_t)(c0 + c) * d + e];
            double* oe = &O[(int64_t)r * d + e];
            *oe = alpha[r] * (*oe) + acc;
          }
        }
      }
      if (tapped) {
        tap->hit = 1;
        memcpy(tap->q1, q1, (size_t)nr * d);
        tap->s_q[0] = sq;
        for (int32_t r = 0; r < nr; ++r) {
          tap->m_new[r] = m[r];
          for (int32_t c = 0; c < nc; ++c) {
            tap->s_int[(int64_t)r * bc + c] = sint[(int64_t)r * bc + c];
            tap->p_tilde[(int64_t)r * bc + c] = pt[(int64_t)r * nc + c];
            tap->p_codes[(int64_t)r * bc + c] = pc[(int64_t)r * nc + c];
          }
          for (int32_t e = 0; e < d; ++e) tap->pv_int[(int64_t)r * d + e] = pv[(int64_t)r * d + e];
        }
        tap->s_p[0] = sp;
      }
    }
    /* O_i = diag(l)^-1 O, L_i = m + log(l). */
    for (int32_t r = 0; r < nr; ++r) {
      for (int32_t e = 0; e < d; ++e)
        o[(int64_t)(r0 + r) * d + e] = (float)(O[(int64_t)r * d + e] / l[r]);
      lse[r0 + r] = (float)((double)m[r] + log(l[r]));
    }
  }
  free(q1); free(x); free(sint); free(pt); free(pc);
  free(pv); free(O); free(l); free(alpha); free(m); free(active); free(sp_row);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Algorithm 2: TurboAttention decode, one query head            */
/* ------------------------------------------------------------------------ */

/* Attends one query to cache blocks [blk_begin, blk_end) and, if with_buffer,
 * then the INT8 buffer block (R-23: explicit split ranges).  k_raw / v_raw are
 * only read under the exact-mode switch (quant = 0): block j = raw tokens
 * [j B_c, (j+1) B_c), buffer = [n_blocks B_c, n_raw).  An empty range returns
 * O = 0, L = -inf (identity element of the combine). */
int32_t tq_decode_head(const tq_params* p, const float* q, const tq_slot* ks, const tq_slot* vs,
                       const float* k_raw, const float* v_raw, int32_t n_raw,
                       int32_t blk_begin, int32_t blk_end, int32_t with_buffer,
                       float* o, float* lse, tq_decode_tap* tap) {
  const int32_t d = p->d, bc = p->block_kv;
  if (!p->quant && (int64_t)ks->n_blocks * bc + ks->n_buf > n_raw) return -1;
  int8_t* q1 = (int8_t*)malloc((size_t)d);
  int8_t* kh = (int8_t*)malloc((size_t)bc * d);
  int8_t* vh = (int8_t*)malloc((size_t)bc * d);
  float* x = (float*)malloc(sizeof(float) * bc);
  int32_t* sint = (int32_t*)malloc(sizeof(int32_t) * bc);
  float* pt = (float*)malloc(sizeof(float) * bc);
  uint8_t* pc = (uint8_t*)malloc((size_t)bc);
  int32_t* pv = (int32_t*)malloc(sizeof(int32_t) * d);
  double* O = (double*)calloc((size_t)d, sizeof(double));
  float sq = 0.0f, m = -INFINITY;
  double l = 0.0;
  if (p->quant) tq_quant_sym8(q, d, q1, &sq);            /* s_Q, Q^q1 */
  sq = st1(p, sq);
  const int32_t n_tiles = (blk_end - blk_begin) + ((with_buffer && ks->n_buf > 0) ? 1 : 0);
  for (int32_t t = 0; t < n_tiles; ++t) {
    const int32_t is_buf = blk_begin + t >= blk_end;
    const int32_t j = is_buf ? -1 : blk_begin + t;
    const int32_t nc = is_buf ? ks->n_buf : bc;
    float s_k, s_v;
    if (p->quant) {
      /* K^q1 = K^q2 s^int + z^int, V likewise; buffer is INT8. */
      for (int32_t c = 0; c < nc; ++c)
        for (int32_t e = 0; e < d; ++e) {
          int64_t ie = (int64_t)c * d + e;
          if (is_buf) {
            kh[ie] = ks->buf[ie];
            vh[ie] = vs->buf[ie];
          } else {
            int64_t cb = (int64_t)j * bc * d + ie, sb = (int64_t)j * d + e;
            kh[ie] = (int8_t)tq_dequant_q2(ks->codes[cb], ks->s_int[sb], ks->z_int[sb]);
            vh[ie] = (int8_t)tq_dequant_q2(vs->codes[cb], vs->s_int[sb], vs->z_int[sb]);
          }
        }
      s_k = is_buf ? st1(p, ks->a_univ / TQ_DIV) : ks->s_parent[j];
      s_v = is_buf ? st1(p, vs->a_univ / TQ_DIV) : vs->s_parent[j];
    } else {
      s_k = s_v = 0.0f;
    }
    const int64_t raw0 = (int64_t)(is_buf ? ks->n_blocks : j) * bc;
    /* S_j = s_Q s_K Q^q1 K_j^q1^T, scaled by 1/sqrt(d) (R-18). */
    const float cqk = (sq * s_k) * p->softmax_scale;
    for (int32_t c = 0; c < nc; ++c) {
      if (p->quant) {
        int32_t acc = 0;
        for (int32_t e = 0; e < d; ++e) acc += (int32_t)q1[e] * (int32_t)kh[(int64_t)c * d + e];
        sint[c] = acc;
        x[c] = (float)acc * cqk;
      } else {
        double acc = 0.0;
        for (int32_t e = 0; e < d; ++e) acc += (double)q[e] * (double)k_raw[(raw0 + c) * d + e];
        sint[c] = 0;
        x[c] = (float)(acc * (double)p->softmax_scale);
      }
    }
    double alpha;
    row_step(p, nc, x, &m, &l, pt, &alpha);
    float sp = 0.0f;
    if (p->quant) {
      const uint8_t row_active = 1;
      sp = quant_p(nc, pt, &row_active, nc, pc);          /* per-row P scale (R-17) */
      for (int32_t e = 0; e < d; ++e) {
        int32_t acc = 0;
        for (int32_t c = 0; c < nc; ++c) acc += (int32_t)pc[c] * (int32_t)vh[(int64_t)c * d + e];
        pv[e] = acc;
      }
      const float cpv = sp * s_v;
      for (int32_t e = 0; e < d; ++e) O[e] = alpha * O[e] + (double)(cpv * (float)pv[e]);
    } else {
      for (int32_t e = 0; e < d; ++e) {
        double acc = 0.0;
        for (int32_t c = 0; c < nc; ++c) acc += (double)pt[c] * (double)v_raw[(raw0 + c) * d + e];
        O[e] = alpha * O[e] + acc;
      }
    }
    if (tap && tap->j_block == j) {
      tap->hit = 1;
      memcpy(tap->q1, q1, (size_t)d);
      tap->s_q[0] = sq;
      tap->m_new[0] = m;
      tap->s_p[0] = sp;
      for (int32_t c = 0; c < nc; ++c) {
        tap->s_int[c] = sint[c];
        tap->p_tilde[c] = pt[c];
        tap->p_codes[c] = pc[c];
      }
      for (int32_t e = 0; e < d; ++e) tap->pv_int[e] = pv[e];
    }
  }
  /* O = diag(l)^-1 O, L = m + log l. */
  if (n_tiles == 0 || l == 0.0) {
    for (int32_t e = 0; e < d; ++e) o[e] = 0.0f;
    *lse = -INFINITY;
  } else {
    for (int32_t e = 0; e < d; ++e) o[e] = (float)(O[e] / l);
    *lse = (float)((double)m + log(l));
  }
  free(q1); free(kh); free(vh); free(x); free(sint); free(pt); free(pc); free(pv); free(O);
  return 0;
}

/* Split-KV combine (R-23): L = max_s L_s + log sum_s e^{L_s - max}, O =
 * sum_s e^{L_s - L} O_s; parts in ascending split order. */
void tq_combine(int32_t n_parts, int32_t d, const float* o_parts, const float* lse_parts,
                float* o, float* lse) {
  double lmax = -INFINITY;
  for (int32_t s = 0; s < n_parts; ++s) lmax = fmax(lmax, (double)lse_parts[s]);
  if (lmax == -INFINITY) {
    for (int32_t e = 0; e < d; ++e) o[e] = 0.0f;
    *lse = -INFINITY;
    return;
  }
  double w_sum = 0.0;
  for (int32_t s = 0; s < n_parts; ++s) w_sum += exp((double)lse_parts[s] - lmax);
  for (int32_t e = 0; e < d; ++e) {
    double acc = 0.0;
    for (int32_t s = 0; s < n_parts; ++s)
      acc += exp((double)lse_parts[s] - lmax) / w_sum * (double)o_parts[(int64_t)s * d + e];
    o[e] = (float)acc;
  }
  *lse = (float)(lmax + log(w_sum));
}

/* Eq. 2: S = QK^T, P = softmax(S scale), H = PV, all in double.
 * Query row r sits at position q_offset + r; causal keeps keys c <= q_offset + r. */
void tq_reference_attention(int32_t nq, int32_t nk, int32_t d, const double* q, const double* k,
                            const double* v, int32_t causal, int32_t q_offset, double scale,
                            double* o, double* lse) {
  double* s = (double*)malloc(sizeof(double) * (nk > 0 ? nk : 1));
  for (int32_t r = 0; r < nq; ++r) {
    int32_t kmax = causal ? q_offset + r + 1 : nk;
    if (kmax > nk) kmax = nk;
    double mx = -INFINITY;
    for (int32_t c = 0; c < kmax; ++c) {
      double acc = 0.0;
      for (int32_t e = 0; e < d; ++e) acc += q[(int64_t)r * d + e] * k[(int64_t)c * d + e];
      s[c] = acc * scale;
      if (s[c] > mx) mx = s[c];
    }
    double sum = 0.0;
    for (int32_t c = 0; c < kmax; ++c) {
      s[c] = exp(s[c] - mx);
      sum += s[c];
    }
    for (int32_t e = 0; e < d; ++e) {
      double acc = 0.0;
      for (int32_t c = 0; c < kmax; ++c) acc += s[c] * v[(int64_t)c * d + e];
      o[(int64_t)r * d + e] = acc / sum;
    }
    lse[r] = mx + log(sum);
  }
  free(s);
}

/* priority = gap * std: gap = max - min over all channels of the
 * head, std = population standard deviation of the per-channel gaps. */
void tq_head_priority(int32_t n, int32_t d, const float* x, double* priority) {
  double* g = (double*)malloc(sizeof(double) * d);
  double gmax = -INFINITY, gmin = INFINITY;
  for (int32_t c = 0; c < d; ++c) {
    double mx = -INFINITY, mn = INFINITY;
    for (int32_t t = 0; t < n; ++t) {
      double v = x[(int64_t)t * d + c];
      if (v > mx) mx = v;
      if (v < mn) mn = v;
    }
    g[c] = mx - mn;
    if (mx > gmax) gmax = mx;
    if (mn < gmin) gmin = mn;
  }
  double mean = 0.0;
  for (int32_t c = 0; c < d; ++c) mean += g[c];
  mean /= d;
  double var = 0.0;
  for (int32_t c = 0; c < d; ++c) var += (g[c] - mean) * (g[c] - mean);
  var /= d;
  *priority = (gmax - gmin) * sqrt(var);
  free(g);
}
