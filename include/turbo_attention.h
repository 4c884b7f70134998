/*
 * turbo_attention.h -- C-ABI of the B200 (sm_100a) TurboAttention hot path
 * (arXiv 2412.08585: FlashQ block-progressive quantisation + SAS softmax).
 *
 * Citations: "P:n" = line n of the paper text with its section /
 * algorithm; "R-n" = reading n in DESIGN.md §3 (where the paper is silent,
 * ambiguous or garbled).
 *
 * Conventions for every entry point
 *   * All tensor pointers are caller-owned DEVICE memory (e.g. torch tensors)
 *     unless the argument says HOST.  The library never allocates or frees,
 *     keeps no mutable global state (beyond one-time caches of device
 *     attributes: SM count, kernel occupancy, the tensor-map encoder entry
 *     point -- one device per process), and never synchronises: work is
 *     enqueued on `stream` (0 = legacy default stream) and completes
 *     asynchronously.
 *   * Developer knobs (environment; results are unchanged): TURBO_QUANT_NOTMA=1
 *     makes turbo_quantize_kv use its per-block fallback kernel instead of the
 *     persistent TMA kernel; TURBO_PREFILL_QPF=n sets the prefill's L2 prefetch
 *     of the next wave's Q rows to n quarter-waves ahead (0 = off).
 *   * Arguments are validated on the host before any launch.  Errors:
 *       TURBO_ERR_INVALID_ARG  null pointer, non-positive size, bad enum value;
 *       TURBO_ERR_UNSUPPORTED  head_dim not in {64,128}, block_kv not in {64,128},
 *                              block_q not in {64,128}, Hq % Hkv != 0,
 *                              sas_nr not in [-30,-1];
 *       TURBO_ERR_CAPACITY     an append/prefill would exceed cache->max_blocks;
 *       TURBO_ERR_CUDA         a CUDA launch failed (cudaGetLastError).
 *     On error nothing has been enqueued (except TURBO_ERR_CUDA, where earlier
 *     kernels of the same call may have run).  No C++ exception crosses the ABI.
 *   * Inputs must be contiguous in the documented layouts and 16-byte aligned.
 *   * The product path has no CPU fallback: without an sm_100 device every
 *     compute call returns TURBO_ERR_CUDA.
 */
#ifndef TURBO_ATTENTION_H
#define TURBO_ATTENTION_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define TURBO_API __attribute__((visibility("default")))
#else
#define TURBO_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TURBO_OK = 0,
  TURBO_ERR_INVALID_ARG = 1,
  TURBO_ERR_UNSUPPORTED = 2,
  TURBO_ERR_CAPACITY = 3,
  TURBO_ERR_CUDA = 4
} turbo_status_t;

typedef void* turbo_stream_t; /* a cudaStream_t */

/* Method parameters (paper defaults: B_r = B_c = n_b = 64, n_r = -6). */
typedef struct {
  int32_t head_dim;      /* d_H in {64, 128} (Eq. 1) */
  int32_t block_q;       /* B_r in {64, 128}: Q stage-1 block rows and P-scale tile rows (Alg. 1) */
  int32_t block_kv;      /* B_c = n_b in {64 (default), 128 (the block-size ablation, Table 3
                            P:758-779)}: K/V stage-1 block, Q2 group length, buffer size, prefill key
                            tile; must equal the cache's block_kv */
  int32_t sas_nr;        /* n_r in [-30, -1]; SAS(x) = 0 for x - m < n_r */
  int32_t alpha_mode;    /* 0: alpha = SAS(m_prev - m_new) literally (Alg. 1, R-15);
                            1: alpha = 1 when the running max is unchanged */
  float softmax_scale;   /* 1/sqrt(d_H) (Eq. 1; R-18) */
  int32_t p_scale_rows;  /* prefill P-scale granularity: 0 = per B_r x B_c tile (Alg. 1, default);
                            1 = per query row x B_c block, as Alg. 2 does -- NEXT-2 variant,
                            oracle flag p_row.  The decode is always per row. */
  int32_t scale_fp16;    /* 0 (default): first-stage scales in FP32 (R-4); 1: every stage-1 scale -- Q, K, V
                            blocks, decode q, parent scales, s_univ -- rounded to binary16 (nearest even)
                            before it is stored or used, as the paper stores them; codes unchanged
                            (R-29) -- NEXT-2 variant, oracle flag scale_fp16.  Must match the value the
                            cache was built with. */
  int32_t sas_fp16;      /* 0 (default): SAS polynomial in binary32 (R-13); 1: the fraction and the
                            coefficients rounded to binary16 and Horner with binary16 FMAs, as the paper
                            evaluates it "in FP16"; LUT factor and product in binary32; used for
                            P~ and alpha in prefill and decode (R-30) -- NEXT-2 variant, oracle flag
                            sas_fp16. */
  void* debug_tap;       /* NULL, or a turbo_debug_tap_t* (see below) */
} turbo_params_t;

/* Paged-free, caller-owned compressed KV cache for ONE layer (P:448-453,
 * P:922-932).  slot = (b, kv_head, kind) with kind 0 = K, 1 = V.  All arrays
 * are device memory sized by turbo_cache_sizes().
 *
 *   block_rec  uint8  [B][Hkv][2][max_blocks][rec_bytes]   one record per flushed
 *              Q2 block: s_int u8[d] | z_int i8[d] | packed codes (see
 *              DESIGN.md §6 "cache layout": K token-major, V channel-major with
 *              a fixed token permutation per 64-token sub-block -- B_c = 128
 *              blocks hold two sub-blocks back to back; 2-bit records use the
 *              first half of the code area).  rec_bytes = 2 d + B_c d / 2.
 *   s_parent   f32    [B][Hkv][2][max_blocks]   first-stage scale of the block
 *   buf        int8   [B][Hkv][2][B_c * d]      INT8 decode buffer (universal
 *              scale): K token-major [t][c], V channel-major [c][t]
 *   a_univ     f32    [B][Hkv][2]               universal max-abs (R-9)
 *   counters   int32  [B][2]                    (n_blocks, n_buf) per sequence
 *   bits       int32  [Hkv][2]  HOST and device copy: 2 or 4 per slot (head-wise
 *              mixed precision P:430-436; R-8)
 * n_tokens / max_blocks are HOST fields maintained by turbo_quantize_kv; all
 * sequences of the batch have the same length. */
typedef struct {
  int32_t batch;
  int32_t n_kv_heads;
  int32_t head_dim;
  int32_t block_kv;
  int32_t max_blocks;
  int64_t n_tokens;            /* HOST mirror of the cached length */
  const int32_t* bits_host;    /* HOST [Hkv][2] */
  const int32_t* bits_dev;     /* device [Hkv][2] */
  uint8_t* block_rec;
  float* s_parent;
  int8_t* buf;
  float* a_univ;
  int32_t* counters;
} turbo_kv_cache_t;

/* Optional debug tap: records the exact-set intermediates of ONE tile so tests
 * can compare them bit-for-bit with the oracle.  Prefill: query head `head`,
 * 64-row Q block `i_block`, KV block `j_block`.  Decode: query head `head`,
 * split 0, block `j_block` (-1 = buffer block).  All pointers device memory. */
typedef struct {
  int32_t batch, head, i_block, j_block;
  int8_t* q1;        /* [64][d] prefill, [d] decode */
  float* s_q;        /* [1] */
  int32_t* s_int;    /* [64][B_c] prefill, [B_c] decode */
  float* m_new;      /* [64] / [1] */
  uint8_t* p_codes;  /* [64][B_c] / [B_c] */
  float* s_p;        /* [1] */
  int32_t* pv_int;   /* [64][d] / [d] */
} turbo_debug_tap_t;

/* Library version and the compiled target ("sm_100a"). */
TURBO_API const char* turbo_version(void);

/* Bytes of each cache array for the given geometry (HOST outputs, any may be NULL). */
TURBO_API turbo_status_t turbo_cache_sizes(int32_t batch, int32_t n_kv_heads, int32_t head_dim, int32_t block_kv,
                                 int32_t max_blocks, size_t* block_rec_bytes, size_t* s_parent_bytes,
                                 size_t* buf_bytes, size_t* a_univ_bytes, size_t* counters_bytes);

/* FlashQ quantisation of K and V into the cache (Alg. 1 P:907-932,
 * Sec. 3.3).
 *   mode 0 = PREFILL: k, v are FP16 [B][n_tokens][Hkv][d].  Resets the cache.
 *     Every B_c block of each (b, kv_head) is quantised to symmetric INT8
 *     (stage 1, s = max|x|/119, code = round_half_even(x * (119/max|x|)));
 *     full blocks are progressively quantised (stage 2: channelwise asymmetric
 *     INT4/INT2 at that slot's bits, integer only) into block records with the
 *     stage-1 scale as parent scale; the n_tokens mod B_c tail is re-quantised
 *     with the universal scale into the INT8 buffer.  The stage-1 operands of
 *     turbo_attention_prefill are written to
 *       k1_out   FP16 [B][Hkv][n_tokens][d]: K's stage-1 codes (integers in [-119,119], exact
 *                in FP16 -- the B operand of the prefill's kind::f16 Q K^T MMA)
 *       v1t_out  FP16 [B][Hkv][T_c][d][B_c]  the stage-1 V codes (integers in
 *                [-119,119], exact in FP16), each block transposed; tokens past
 *                n_tokens are 0; T_c = ceil(n_tokens / B_c)
 *       k1_scale_out, v1_scale_out  f32 [B][Hkv][T_c].
 *   mode 1 = APPEND: k, v are FP16 [B][Hkv][d] (one new token per sequence,
 *     n_tokens must be 1).  Quantised with the universal scale and clamped to
 *     +-119 into the buffer; a full buffer (n_b = B_c tokens) is flushed to a
 *     stage-2 block with parent scale a_univ/119.  The *_out pointers must be
 *     NULL.  Updates cache->n_tokens (host) and the device counters.
 *   mode 2 = PREFILL_CHUNK (R-28, R-31, NEXT-3): k, v FP16 [B][n_tokens][Hkv][d],
 *     a further prefill chunk after the P = cache->n_tokens cached tokens.  When
 *     P is not a whole number of blocks (R-31) the chunk's first
 *     min(n_tokens, B_c - P % B_c) tokens complete the buffered block exactly
 *     as APPEND does (universal scale, clamp, flush with parent a_univ/119);
 *     their stage-1 outputs are those codes (the block's scale comes from
 *     turbo_dequantize_cache).  The rest of the chunk is block-aligned: the
 *     universal scales become the running max over it and the previous value,
 *     its full blocks are appended, its tail goes to the buffer.
 *     The stage-1 outputs cover Nk = P + n_tokens tokens (k1_out
 *     [B][Hkv][Nk][d], v1t_out [B][Hkv][ceil(Nk/B_c)][d][B_c], scales
 *     [B][Hkv][ceil(Nk/B_c)]); the chunk's are written at token P / block
 *     P / B_c (the prefix part comes from turbo_dequantize_cache).  Updates
 *     cache->n_tokens to Nk. */
TURBO_API turbo_status_t turbo_quantize_kv(const turbo_params_t* params, turbo_kv_cache_t* cache, const void* k,
                                 const void* v, int32_t n_tokens, int32_t mode, void* k1_out,
                                 void* v1t_out, float* k1_scale_out, float* v1_scale_out,
                                 turbo_stream_t stream);

/* Algorithm 1, TurboAttention prefill, tcgen05 INT8 MMA.
 *   q       FP16 [B][N][Hq][d]; quantised per B_r x d block inside the kernel.
 *   k1, v1t, k1_scale, v1_scale: the stage-1 operands from turbo_quantize_kv
 *           (same B, N, Hkv, params).
 *   causal  1 = key <= query (R-20), 0 = full.
 *   o       FP16 [B][N][Hq][d] = O_i / l, round to nearest even.
 *   lse     f32 [B][Hq][N] = m + ln l.
 * Query head h reads kv head h / (Hq/Hkv) (GQA, R-22). */
TURBO_API turbo_status_t turbo_attention_prefill(const turbo_params_t* params, int32_t B, int32_t N, int32_t Hq,
                                       int32_t Hkv, int32_t causal, const void* q, const void* k1,
                                       const void* v1t, const float* k1_scale, const float* v1_scale,
                                       void* o, float* lse, turbo_stream_t stream);

/* The Q projection with the stage-1 Q quantisation fused into its epilogue (Sec. 5: "we
 * fused the QKV projection with quantization"; NEXT-3), tcgen05 kind::f16 GEMM:
 *   x       FP16 [B][N][D] (the layer input, token-major), D % 64 == 0.
 *   wq      FP16 [Hq * d][D] (one row per output feature); (Hq * d) % 256 == 0.
 *   q1_out  INT8 [B][N][Hq][d]: Q^q1 of Q = fp16(x wq^T) (the projection's FP16 output, rounded to
 *           nearest even), stage 1 per (b, head, B_r-row block) exactly as turbo_attention_prefill
 *           does it (Alg. 1; R-2, R-3; scale_fp16: R-29).
 *   sq_out  f32 [B][Hq][ceil(N / B_r)] the blocks' scales.
 *   q16_out FP16 [B][N][Hq][d] (the unquantised projection, for checking) or NULL.
 * Errors: TURBO_ERR_UNSUPPORTED for D % 64 != 0 or (Hq d) % 256 != 0. */
TURBO_API turbo_status_t turbo_q_projection(const turbo_params_t* params, int32_t B, int32_t N, int32_t D, int32_t Hq,
                                            const void* x, const void* wq, int8_t* q1_out, float* sq_out,
                                            void* q16_out, turbo_stream_t stream);

/* turbo_attention_prefill with the query already quantised (q1 INT8 [B][N][Hq][d] and q1_scale
 * f32 [B][Hq][ceil(N / B_r)], e.g. from turbo_q_projection): identical results to
 * turbo_attention_prefill on the FP16 Q those codes came from; the kernel reads d instead of 2d
 * bytes per query row. */
TURBO_API turbo_status_t turbo_attention_prefill_q1(const turbo_params_t* params, int32_t B, int32_t N, int32_t Hq,
                                                    int32_t Hkv, int32_t causal, const int8_t* q1,
                                                    const float* q1_scale, const void* k1, const void* v1t,
                                                    const float* k1_scale, const float* v1_scale, void* o, float* lse,
                                                    turbo_stream_t stream);

/* Stage-1 reconstruction of flushed cache blocks [blk_begin, blk_end)
 * (blk_end = -1: all; blocks past a sequence's count are skipped), the
 * prefix operands of a chunked prefill (R-28): k1_out FP16 [B][Hkv][Nk][d] rows
 * [B_c j, B_c j + B_c) and v1t_out [B][Hkv][ceil(Nk/B_c)][d][B_c] block j get
 * code s_int + z_int (Alg. 2), the scales the blocks' parent
 * scales.  With blk_end = -1 and buffered tokens (R-31) these follow as block
 * n_blocks: their INT8 codes, scale a_univ/119, the block's later v1t columns
 * zero.  Nk = token capacity of k1_out (>= B_c x the last block, and >= the
 * cached length when the buffer is written).  The cache is not modified. */
TURBO_API turbo_status_t turbo_dequantize_cache(const turbo_params_t* params, const turbo_kv_cache_t* cache,
                                                int32_t blk_begin, int32_t blk_end, void* k1_out, void* v1t_out,
                                                float* k1_scale_out, float* v1_scale_out, int32_t Nk,
                                                turbo_stream_t stream);

/* Chunked prefill (NEXT-3, reading R-28): Algorithm 1 for Nq new queries at
 * absolute positions [Nk - Nq, Nk) against Nk keys, e.g. a compressed-cache
 * prefix of Nk - Nq tokens (its stage-1 reconstruction from
 * turbo_dequantize_cache) followed by the chunk's own keys (turbo_quantize_kv
 * mode 2).  turbo_attention_prefill is the case Nq = Nk.
 *   q       FP16 [B][Nq][Hq][d];  k1 FP16 codes [B][Hkv][Nk][d];
 *   v1t     FP16 codes [B][Hkv][T_k][d][B_c], T_k = ceil(Nk / B_c);
 *   k1_scale, v1_scale  f32 [B][Hkv][T_k];
 *   causal  1 = key <= Nk - Nq + query row, 0 = all Nk keys;
 *   o       FP16 [B][Nq][Hq][d];  lse f32 [B][Hq][Nq].
 * Errors: TURBO_ERR_INVALID_ARG if Nq < 1 or Nk < Nq. */
TURBO_API turbo_status_t turbo_attention_prefill_chunk(const turbo_params_t* params, int32_t B, int32_t Nq,
                                                       int32_t Nk, int32_t Hq, int32_t Hkv, int32_t causal,
                                                       const void* q, const void* k1, const void* v1t,
                                                       const float* k1_scale, const float* v1_scale, void* o,
                                                       float* lse, turbo_stream_t stream);

/* Workspace for turbo_attention_decode with n_splits on the current device
 * (HOST result; 0 = none needed, or invalid arguments).
 *   n_splits >= 2: S * B * Hq * (d + 1) floats;  n_splits <= 0 (balanced):
 *   (B * Hkv' + W) * (Hq / Hkv') * (d + 1) floats, W = -n_splits, or
 *   turbo_decode_workers() for n_splits == 0; Hkv' = Hkv * r (see below). */
TURBO_API size_t turbo_decode_workspace_bytes(int32_t B, int32_t Hq, int32_t Hkv, int32_t head_dim,
                                              int32_t n_splits);

/* Worker warps W of the balanced decode schedule on the current device
 * (every SM filled to the decode kernel's occupancy; HOST result, 0 if no
 * device).  Exposed so that callers can reproduce the partition below. */
TURBO_API int32_t turbo_decode_workers(int32_t Hq, int32_t Hkv, int32_t head_dim);

/* Algorithm 2, TurboAttention decode of one new query per
 * sequence against cache blocks [blk_begin, blk_end) (blk_end = -1: all
 * flushed blocks) and, if with_buffer, the INT8 buffer block last.  Each
 * sub-range below is one online-softmax pass (same order as Alg. 2); the
 * partial results are merged by the log-sum-exp combine (R-23; fixed
 * summation order, see turbo_combine_lse).  Sub-ranges:
 *   n_splits in [1, 12000]: the block range of every (b, kv head) is cut into
 *     n_splits contiguous ranges of ceil(n / n_splits) blocks (the buffer
 *     joins the last one).
 *   n_splits in [-12000, 0] (balanced): the units of every (b, kv head) --
 *     its blocks in order, then the buffer block if used (with_buffer and
 *     n_buf > 0) -- are laid end to end in (b, kv head) order (GQA groups of
 *     G > 8 query rows: each KV head counts as r virtual heads of G / r rows,
 *     r the least divisor of G with G / r <= 8, in (kv head, row group) order); the sequence
 *     of all `total` units is cut into chunks of C = max(8, ceil(total / W))
 *     units, W = -n_splits workers, or W = turbo_decode_workers(Hq, Hkv, d)
 *     (the current device's resident decode warps) for n_splits == 0, and
 *     every (b, kv head) range is split at the chunk boundaries.  Every warp
 *     streams the same number of bytes, whatever the lengths of the sequences.
 * SPLIT DEPENDENCE: the result is a deterministic function of the inputs and
 * of the sub-range partition, but it DEPENDS on the partition: each pass has
 * its own running max, alpha chain and per-row P scales, so a
 * split decode is not bit-identical to the unsplit Alg. 2 (n_splits = 1); the
 * size of the difference is reported by bench.py (`deviation.decode_split`,
 * both alpha modes).  Every n_splits != 0 gives a device-independent
 * partition; n_splits == 0 follows the device's SM count and occupancy, so its
 * numbers can differ between GPUs (the Python binding's default therefore
 * passes an explicit worker count, never 0).
 *   q      FP16 [B][Hq][d]; quantised per (b, head) vector.
 *   workspace  device, >= turbo_decode_workspace_bytes(B, Hq, Hkv, d, n_splits).
 *   o      FP16 [B][Hq][d] or NULL;  o_part f32 [B][Hq][d] (normalised) or
 *          NULL -- at least one of them;  lse f32 [B][Hq] (required).
 * Empty range with no buffer tokens: o = 0, lse = -inf. */
TURBO_API turbo_status_t turbo_attention_decode(const turbo_params_t* params, const turbo_kv_cache_t* cache,
                                      int32_t Hq, const void* q, int32_t blk_begin, int32_t blk_end,
                                      int32_t with_buffer, int32_t n_splits, void* workspace,
                                      size_t workspace_bytes, void* o, float* o_part, float* lse,
                                      turbo_stream_t stream);

/* Log-sum-exp combine of n_parts partial results (R-23):
 * L = max_s L_s + ln sum_s e^{L_s - max}, O = sum_s e^{L_s - L} O_s.
 * Deterministic fixed summation order: the weight sum lane-strided then by
 * butterfly; O over W <= 8 contiguous part ranges (about 4 parts per range),
 * each ascending, the ranges added in order.  n_parts <= 12000.
 *   d = head_dim (64 or 128, else TURBO_ERR_UNSUPPORTED);
 *   o_parts f32 [n_parts][rows][d], lse_parts f32 [n_parts][rows];
 *   o FP16 [rows][d] (or NULL), o_f32 f32 [rows][d] (or NULL), lse f32 [rows]. */
TURBO_API turbo_status_t turbo_combine_lse(int32_t n_parts, int32_t rows, int32_t d, const float* o_parts,
                                 const float* lse_parts, void* o, float* o_f32, float* lse,
                                 turbo_stream_t stream);

/* Head-wise mixed precision planner (Sec. 3.2; R-8).
 * turbo_head_priority: for every slot (kv_head h, kind K=0 / V=1) over all
 *   B x N prefill tokens of k, v (FP16 [B][N][Hkv][d]):
 *   priority[h][kind] = (max_c max_t x - min_c min_t x) * std_c(max_t x_c - min_t x_c)
 *   (population std over the d channel gaps), written as f64 to device memory.
 *   workspace: device, >= turbo_priority_workspace_bytes(Hkv, d).
 * turbo_plan_bits (HOST): the n_2bit lowest-priority slots get 2 bits, the
 *   others 4; ties go to the lower slot index (slot = 2 h + kind). */
TURBO_API size_t turbo_priority_workspace_bytes(int32_t n_kv_heads, int32_t head_dim);
TURBO_API turbo_status_t turbo_head_priority(int32_t B, int32_t N, int32_t Hkv, int32_t head_dim, const void* k,
                                             const void* v, void* workspace, size_t workspace_bytes,
                                             double* priority, turbo_stream_t stream);
TURBO_API turbo_status_t turbo_plan_bits(const double* priority, int32_t n_slots, int32_t n_2bit, int32_t* bits);

/* Self-test (not on the hot path): compares the library's fast correctly
 * rounded divisions used for the stage-1 and P scales (which = 0: a / 119,
 * which = 1: 119 / a; Alg. 1, Alg. 2) with IEEE
 * division for every binary32 bit pattern in [lo_bits, hi_bits].  Adds the
 * number of mismatches to *mismatches (device u64) and lowers *first_bad
 * (device u32) to the smallest mismatching pattern.  Async on the stream. */
TURBO_API turbo_status_t turbo_selftest_div(int32_t which, uint32_t lo_bits, uint32_t hi_bits,
                                            unsigned long long* mismatches, uint32_t* first_bad,
                                            turbo_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* TURBO_ATTENTION_H */
