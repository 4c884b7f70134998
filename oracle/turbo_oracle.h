/*
 * turbo_oracle.h -- CPU oracle for TurboAttention (arXiv 2412.08585).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2412_08585_b200/, include/turbo_attention.h) never links or calls it,
 * and the two share no code, headers, tables or constants.
 *
 * Citation convention: "P:n" = line n of the paper text, with the
 * section / equation / algorithm it falls in; "R-n" = reading n in DESIGN.md §3
 * (where the paper is silent, ambiguous or garbled).
 *
 * Every function follows the paper's algorithm step by step (Alg. 1 P:885-941,
 * Alg. 2, SAS P:455-493 and Appendix B), plain scalar C,
 * no blocking or reordering beyond what those algorithms state.
 */
#ifndef TURBO_ORACLE_H
#define TURBO_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t d;             /* head dim d_H (Eq. 1) */
  int32_t block_q;       /* B_r (Alg. 1) */
  int32_t block_kv;      /* B_c = n_b */
  int32_t sas_nr;        /* n_r, negative integer */
  int32_t alpha_mode;    /* 0: alpha = SAS(m_new - m_prev) literally; 1: alpha=1 if max unchanged (R-15) */
  float softmax_scale;   /* 1/sqrt(d_H) (Eq. 1; R-18) */
  int32_t quant;         /* 1: FlashQ quantization as in Alg. 1/2; 0: exact-mode switch (pin P5) */
  int32_t sas;           /* 1: SAS exponent; 0: exact exp (pin P5) */
  int32_t p_row;         /* prefill P scale: 0 per B_r x B_c tile (Alg. 1); 1 per row x B_c block,
                            the granularity Alg. 2 uses -- NEXT-2 variant */
  int32_t scale_fp16;    /* first-stage scales stored in FP16 (Eq. 8 text): every stage-1 scale
                            s = max|x|/119 (Q, K, V blocks, decode q, parent scales, s_univ) is rounded to
                            binary16 (nearest even) before use; codes unchanged (R-29) -- NEXT-2 variant */
  int32_t sas_fp16;      /* SAS polynomial in FP16: f and the coefficients rounded to binary16,
                            Horner with binary16 FMAs; LUT and product in binary32 (R-30) -- NEXT-2 variant */
} tq_params;

/* One cache "slot" = one (batch, kv_head, K-or-V) stream.  Logical layout
 * (unpacked): codes[block][token][channel]. */
typedef struct {
  int32_t bits;          /* 2 or 4 (head-wise mixed precision) */
  int32_t max_blocks;
  int32_t n_blocks;      /* flushed Q2 blocks */
  int32_t n_buf;         /* tokens in the INT8 buffer */
  uint8_t* codes;        /* [max_blocks][B_c][d]  values in [0, 2^bits-1] */
  uint8_t* s_int;        /* [max_blocks][d] */
  int8_t* z_int;         /* [max_blocks][d] */
  float* s_parent;       /* [max_blocks]  first-stage (parent) scale of each block */
  int8_t* buf;           /* [B_c][d] INT8 buffer codes */
  float a_univ;          /* universal max-abs (R-9); s_univ = a_univ/119 */
} tq_slot;

/* Trace of one prefill tile (B_r block i, KV block j) -- the "exact set". */
typedef struct {
  int32_t i_block, j_block;
  int32_t hit;           /* set to 1 when the tile was visited */
  int8_t* q1;            /* [B_r][d] */
  float* s_q;            /* [1] */
  int32_t* s_int;        /* [B_r][B_c]; masked entries left 0 */
  float* m_new;          /* [B_r] running max after this tile */
  float* p_tilde;        /* [B_r][B_c] */
  uint8_t* p_codes;      /* [B_r][B_c] */
  float* s_p;            /* [1] */
  int32_t* pv_int;       /* [B_r][d] */
} tq_prefill_tap;

/* Trace of one decode tile (block j, or j = -1 for the buffer block). */
typedef struct {
  int32_t j_block;
  int32_t hit;
  int8_t* q1;            /* [d] */
  float* s_q;            /* [1] */
  int32_t* s_int;        /* [B_c] */
  float* m_new;          /* [1] */
  float* p_tilde;        /* [B_c] */
  uint8_t* p_codes;      /* [B_c] */
  float* s_p;            /* [1] */
  int32_t* pv_int;       /* [d] */
} tq_decode_tap;

/* --- SAS (Sec. 4; Appendix B) --- */
void tq_sas_lut(int32_t nr, float* lut /* [-nr + 1] */);
float tq_sas_poly(float f);
float tq_sas(float dist, int32_t nr);
float tq_sas_poly_fp16(float f);
float tq_sas_fp16(float dist, int32_t nr);
void tq_sas_softmax_rows(int32_t rows, int32_t cols, const float* x, int32_t nr, float* out);

/* --- FlashQ stage 1 / stage 2 (Eq. 9/10; Alg. 1) --- */
void tq_quant_sym8(const float* x, int64_t n, int8_t* codes, float* s_out);
void tq_quant_asym(const int8_t* g, int32_t n, int64_t stride, int32_t bits,
                   uint8_t* codes, int64_t code_stride, uint8_t* s_int, int8_t* z_int);
int32_t tq_dequant_q2(int32_t code, int32_t s_int, int32_t z_int);

/* --- KV cache (Sec. 3.3, Alg. 1) --- */
int32_t tq_cache_prefill_slot(const tq_params* p, int32_t n_tokens, const float* x /*[N][d]*/,
                              tq_slot* slot, int8_t* x1 /*[N][d] or NULL*/,
                              float* x1_scale /*[T_c] or NULL*/);
int32_t tq_cache_append_slot(const tq_params* p, const float* x /*[d]*/, tq_slot* slot);
float tq_slot_univ_scale(const tq_params* p, const tq_slot* slot);

/* --- Attention --- */
int32_t tq_prefill_head(const tq_params* p, int32_t n, int32_t causal, const float* q,
                        const float* k, const float* v, float* o, float* lse,
                        tq_prefill_tap* tap);
int32_t tq_prefill_head_blocks(const tq_params* p, int32_t n, int32_t causal, const float* q,
                               const float* k, const float* v, int32_t i_begin, int32_t i_end,
                               float* o, float* lse, tq_prefill_tap* tap);
/* Chunked prefill (R-28): Alg. 1 for nq queries at positions nk-nq .. nk-1
 * against nk keys given as stage-1 operands (k1, v1 int8 [nk][d], block
 * scales sk, sv); quantisation mode only. */
int32_t tq_prefill_chunk_head(const tq_params* p, int32_t nq, int32_t nk, int32_t causal, const float* q,
                              const int8_t* k1, const float* sk, const int8_t* v1, const float* sv,
                              float* o, float* lse);
int32_t tq_cache_prefill_append_slot(const tq_params* p, int32_t n_tokens, const float* x, tq_slot* s,
                                     int8_t* x1, float* x1_scale);
int32_t tq_decode_head(const tq_params* p, const float* q, const tq_slot* ks, const tq_slot* vs,
                       const float* k_raw, const float* v_raw, int32_t n_raw,
                       int32_t blk_begin, int32_t blk_end, int32_t with_buffer,
                       float* o, float* lse, tq_decode_tap* tap);
void tq_combine(int32_t n_parts, int32_t d, const float* o_parts, const float* lse_parts,
                float* o, float* lse);
void tq_reference_attention(int32_t nq, int32_t nk, int32_t d, const double* q, const double* k,
                            const double* v, int32_t causal, int32_t q_offset, double scale,
                            double* o, double* lse);

/* --- Head-wise mixed precision planner (Sec. 3.2) --- */
void tq_head_priority(int32_t n_tokens, int32_t d, const float* x /*[N][d]*/, double* priority);

#ifdef __cplusplus
}
#endif
#endif
