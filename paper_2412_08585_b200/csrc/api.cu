// api.cu -- extern "C" entry points of libturboattn.so (include/turbo_attention.h):
// host-side validation, then the kernel launchers.  No allocation, no
// synchronisation, no mutable global state.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "layout.cuh"

namespace ta_host {
cudaError_t launch_quant_prefill(const turbo_kv_cache_t* c, const __half* k, const __half* v, int N, __half* k1,
                                 __half* v1t, float* k1s, float* v1s, cudaStream_t st, int j0, int Nk,
                                 int scale_fp16);
cudaError_t launch_dequant_cache(const turbo_kv_cache_t* c, int blk_begin, int blk_end, int Nk, __half* k1,
                                 __half* v1t, float* k1s, float* v1s, cudaStream_t st, int scale_fp16);
cudaError_t launch_quant_append(const turbo_kv_cache_t* c, const __half* k, const __half* v, cudaStream_t st,
                                int scale_fp16);
cudaError_t launch_prefill(const turbo_params_t* p, int B, int N, int Nk, int Hq, int Hkv, int causal, const __half* q,
                           const __half* k1, const __half* v1t, const float* k1s, const float* v1s, __half* o,
                           float* lse, cudaStream_t st, const int8_t* q1_in = nullptr, const float* sq_in = nullptr);
cudaError_t launch_q_projection(const turbo_params_t* p, int B, int N, int D, int Hq, const __half* x, const __half* wq,
                                int8_t* q1, float* sq, __half* q16, cudaStream_t st);
size_t decode_workspace(int B, int Hq, int Hkv, int HD, int S);
int decode_workers(int Hq, int Hkv, int HD);
int decode_row_groups(int G);
cudaError_t launch_decode(const turbo_params_t* p, const turbo_kv_cache_t* c, int Hq, const __half* q, int blk_begin,
                          int blk_end, int with_buffer, int S, void* ws, __half* o, float* o_part, float* lse,
                          cudaStream_t st);
cudaError_t launch_combine(int n_parts, int rows, int d, const float* o_parts, const float* lse_parts, __half* o,
                           float* o32, float* lse, cudaStream_t st);

size_t priority_workspace(int Hkv, int HD);
cudaError_t launch_selftest_div(int which, uint32_t lo, uint32_t hi, unsigned long long* bad, uint32_t* first,
                                cudaStream_t st);
cudaError_t launch_priority(int B, int N, int Hkv, int HD, const __half* k, const __half* v, void* ws,
                            double* priority, cudaStream_t st);
void plan_bits(const double* priority, int n_slots, int n_2bit, int32_t* bits);

// SAS threshold |n_r|; the LUT itself is ta::kExpNegBits.
void fill_sas_const(ta::SasConst* sc, int32_t nr) {
  sc->nr_abs = (float)(-nr);
  sc->nr_int = -nr;
}
}  // namespace ta_host

namespace {
turbo_status_t check_params(const turbo_params_t* p) {
  if (!p) return TURBO_ERR_INVALID_ARG;
  if (p->head_dim != 64 && p->head_dim != 128) return TURBO_ERR_UNSUPPORTED;
  if (p->block_kv != 64 && p->block_kv != 128) return TURBO_ERR_UNSUPPORTED;
  if (p->block_q != 64 && p->block_q != 128) return TURBO_ERR_UNSUPPORTED;
  if (p->sas_nr < -30 || p->sas_nr > -1) return TURBO_ERR_UNSUPPORTED;
  if (p->alpha_mode != 0 && p->alpha_mode != 1) return TURBO_ERR_INVALID_ARG;
  if (!(p->softmax_scale > 0.0f) || !std::isfinite(p->softmax_scale)) return TURBO_ERR_INVALID_ARG;
  if (p->p_scale_rows != 0 && p->p_scale_rows != 1) return TURBO_ERR_INVALID_ARG;
  if (p->scale_fp16 != 0 && p->scale_fp16 != 1) return TURBO_ERR_INVALID_ARG;
  if (p->sas_fp16 != 0 && p->sas_fp16 != 1) return TURBO_ERR_INVALID_ARG;
  return TURBO_OK;
}

turbo_status_t check_cache(const turbo_params_t* p, const turbo_kv_cache_t* c) {
  if (!c) return TURBO_ERR_INVALID_ARG;
  if (c->batch < 1 || c->n_kv_heads < 1 || c->max_blocks < 0) return TURBO_ERR_INVALID_ARG;
  if (c->head_dim != p->head_dim || c->block_kv != p->block_kv) return TURBO_ERR_INVALID_ARG;
  if (!c->bits_host || !c->bits_dev || !c->block_rec || !c->s_parent || !c->buf || !c->a_univ || !c->counters)
    return TURBO_ERR_INVALID_ARG;
  for (int i = 0; i < 2 * c->n_kv_heads; ++i)
    if (c->bits_host[i] != 2 && c->bits_host[i] != 4) return TURBO_ERR_INVALID_ARG;
  return TURBO_OK;
}

turbo_status_t cuda_status(cudaError_t e) { return e == cudaSuccess ? TURBO_OK : TURBO_ERR_CUDA; }
}  // namespace

extern "C" {

const char* turbo_version(void) { return "turboattn 0.1.0 sm_100a"; }

turbo_status_t turbo_cache_sizes(int32_t batch, int32_t n_kv_heads, int32_t head_dim, int32_t block_kv,
                                 int32_t max_blocks, size_t* block_rec_bytes, size_t* s_parent_bytes,
                                 size_t* buf_bytes, size_t* a_univ_bytes, size_t* counters_bytes) {
  if (batch < 1 || n_kv_heads < 1 || max_blocks < 0) return TURBO_ERR_INVALID_ARG;
  if (head_dim != 64 && head_dim != 128) return TURBO_ERR_UNSUPPORTED;
  if (block_kv != 64 && block_kv != 128) return TURBO_ERR_UNSUPPORTED;
  const size_t slots = (size_t)batch * n_kv_heads * 2;
  if (block_rec_bytes) *block_rec_bytes = slots * max_blocks * ta::rec_bytes(head_dim, block_kv);
  if (s_parent_bytes) *s_parent_bytes = slots * max_blocks * sizeof(float);
  if (buf_bytes) *buf_bytes = slots * block_kv * head_dim;
  if (a_univ_bytes) *a_univ_bytes = slots * sizeof(float);
  if (counters_bytes) *counters_bytes = (size_t)batch * 2 * sizeof(int32_t);
  return TURBO_OK;
}

turbo_status_t turbo_quantize_kv(const turbo_params_t* params, turbo_kv_cache_t* cache, const void* k,
                                 const void* v, int32_t n_tokens, int32_t mode, void* k1_out, void* v1t_out,
                                 float* k1_scale_out, float* v1_scale_out, turbo_stream_t stream) {
  turbo_status_t s = check_params(params);
  if (s != TURBO_OK) return s;
  if ((s = check_cache(params, cache)) != TURBO_OK) return s;
  if (!k || !v) return TURBO_ERR_INVALID_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (mode == 0) {
    if (n_tokens < 1 || !k1_out || !v1t_out || !k1_scale_out || !v1_scale_out) return TURBO_ERR_INVALID_ARG;
    if (n_tokens / params->block_kv > cache->max_blocks) return TURBO_ERR_CAPACITY;
    s = cuda_status(ta_host::launch_quant_prefill(cache, reinterpret_cast<const __half*>(k),
                                                  reinterpret_cast<const __half*>(v), n_tokens, reinterpret_cast<__half*>(k1_out),
                                                  reinterpret_cast<__half*>(v1t_out),
                                                  k1_scale_out, v1_scale_out, st, 0, n_tokens,
                                                  params->scale_fp16));
    if (s == TURBO_OK) cache->n_tokens = n_tokens;
    return s;
  }
  if (mode == 2) {  // a further prefill chunk (R-28; R-31 when the cache ends inside a block)
    if (n_tokens < 1 || !k1_out || !v1t_out || !k1_scale_out || !v1_scale_out) return TURBO_ERR_INVALID_ARG;
    if (cache->n_tokens < 1) return TURBO_ERR_INVALID_ARG;
    const int64_t nk = cache->n_tokens + n_tokens;
    if (nk / params->block_kv > cache->max_blocks || nk > INT32_MAX) return TURBO_ERR_CAPACITY;
    s = cuda_status(ta_host::launch_quant_prefill(cache, reinterpret_cast<const __half*>(k),
                                                  reinterpret_cast<const __half*>(v), n_tokens, reinterpret_cast<__half*>(k1_out),
                                                  reinterpret_cast<__half*>(v1t_out), k1_scale_out, v1_scale_out,
                                                  st, (int)(cache->n_tokens / params->block_kv), (int)nk,
                                                  params->scale_fp16));
    if (s == TURBO_OK) cache->n_tokens = nk;
    return s;
  }
  if (mode == 1) {
    if (n_tokens != 1 || k1_out || v1t_out || k1_scale_out || v1_scale_out) return TURBO_ERR_INVALID_ARG;
    if (cache->n_tokens < 1) return TURBO_ERR_INVALID_ARG;  // universal scale comes from a prefill
    if ((cache->n_tokens + 1) / params->block_kv > cache->max_blocks) return TURBO_ERR_CAPACITY;
    s = cuda_status(ta_host::launch_quant_append(cache, reinterpret_cast<const __half*>(k),
                                                 reinterpret_cast<const __half*>(v), st, params->scale_fp16));
    if (s == TURBO_OK) cache->n_tokens += 1;
    return s;
  }
  return TURBO_ERR_INVALID_ARG;
}

turbo_status_t turbo_dequantize_cache(const turbo_params_t* params, const turbo_kv_cache_t* cache,
                                      int32_t blk_begin, int32_t blk_end, void* k1_out, void* v1t_out,
                                      float* k1_scale_out, float* v1_scale_out, int32_t Nk, turbo_stream_t stream) {
  turbo_status_t s = check_params(params);
  if (s != TURBO_OK) return s;
  if ((s = check_cache(params, cache)) != TURBO_OK) return s;
  if (!k1_out || !v1t_out || !k1_scale_out || !v1_scale_out || blk_begin < 0) return TURBO_ERR_INVALID_ARG;
  const int64_t flushed = cache->n_tokens / params->block_kv;
  const int64_t last = blk_end < 0 ? flushed : std::min<int64_t>(blk_end, flushed);
  if (blk_end >= 0 && blk_end < blk_begin) return TURBO_ERR_INVALID_ARG;
  if (Nk < 1 || last * params->block_kv > Nk) return TURBO_ERR_INVALID_ARG;
  // blk_end < 0 with buffered tokens: they are written too, as the boundary block (R-31)
  if (blk_end < 0 && cache->n_tokens % params->block_kv != 0 && cache->n_tokens > Nk) return TURBO_ERR_INVALID_ARG;
  return cuda_status(ta_host::launch_dequant_cache(cache, blk_begin, blk_end, Nk, reinterpret_cast<__half*>(k1_out),
                                                   reinterpret_cast<__half*>(v1t_out), k1_scale_out, v1_scale_out,
                                                   reinterpret_cast<cudaStream_t>(stream), params->scale_fp16));
}

turbo_status_t turbo_attention_prefill_chunk(const turbo_params_t* params, int32_t B, int32_t Nq, int32_t Nk,
                                             int32_t Hq, int32_t Hkv, int32_t causal, const void* q, const void* k1,
                                             const void* v1t, const float* k1_scale, const float* v1_scale, void* o,
                                             float* lse, turbo_stream_t stream) {
  turbo_status_t s = check_params(params);
  if (s != TURBO_OK) return s;
  if (B < 1 || Nq < 1 || Nk < Nq || Hq < 1 || Hkv < 1 || (causal != 0 && causal != 1)) return TURBO_ERR_INVALID_ARG;
  if (Hq % Hkv != 0) return TURBO_ERR_UNSUPPORTED;
  if (!q || !k1 || !v1t || !k1_scale || !v1_scale || !o || !lse) return TURBO_ERR_INVALID_ARG;
  return cuda_status(ta_host::launch_prefill(params, B, Nq, Nk, Hq, Hkv, causal, reinterpret_cast<const __half*>(q),
                                             reinterpret_cast<const __half*>(k1), reinterpret_cast<const __half*>(v1t),
                                             k1_scale, v1_scale,
                                             reinterpret_cast<__half*>(o), lse, reinterpret_cast<cudaStream_t>(stream)));
}

turbo_status_t turbo_q_projection(const turbo_params_t* params, int32_t B, int32_t N, int32_t D, int32_t Hq,
                                  const void* x, const void* wq, int8_t* q1_out, float* sq_out, void* q16_out,
                                  turbo_stream_t stream) {
  turbo_status_t s = check_params(params);
  if (s != TURBO_OK) return s;
  if (B < 1 || N < 1 || D < 64 || Hq < 1) return TURBO_ERR_INVALID_ARG;
  if (D % 64 != 0 || (Hq * params->head_dim) % 256 != 0) return TURBO_ERR_UNSUPPORTED;
  if (!x || !wq || !q1_out || !sq_out) return TURBO_ERR_INVALID_ARG;
  return cuda_status(ta_host::launch_q_projection(params, B, N, D, Hq, reinterpret_cast<const __half*>(x),
                                                  reinterpret_cast<const __half*>(wq), q1_out, sq_out,
                                                  reinterpret_cast<__half*>(q16_out),
                                                  reinterpret_cast<cudaStream_t>(stream)));
}

turbo_status_t turbo_attention_prefill_q1(const turbo_params_t* params, int32_t B, int32_t N, int32_t Hq,
                                          int32_t Hkv, int32_t causal, const int8_t* q1, const float* q1_scale,
                                          const void* k1, const void* v1t, const float* k1_scale,
                                          const float* v1_scale, void* o, float* lse, turbo_stream_t stream) {
  turbo_status_t s = check_params(params);
  if (s != TURBO_OK) return s;
  if (B < 1 || N < 1 || Hq < 1 || Hkv < 1 || (causal != 0 && causal != 1)) return TURBO_ERR_INVALID_ARG;
  if (Hq % Hkv != 0) return TURBO_ERR_UNSUPPORTED;
  if (!q1 || !q1_scale || !k1 || !v1t || !k1_scale || !v1_scale || !o || !lse) return TURBO_ERR_INVALID_ARG;
  return cuda_status(ta_host::launch_prefill(params, B, N, N, Hq, Hkv, causal, nullptr,
                                             reinterpret_cast<const __half*>(k1),
                                             reinterpret_cast<const __half*>(v1t), k1_scale, v1_scale,
                                             reinterpret_cast<__half*>(o), lse, reinterpret_cast<cudaStream_t>(stream),
                                             q1, q1_scale));
}

turbo_status_t turbo_attention_prefill(const turbo_params_t* params, int32_t B, int32_t N, int32_t Hq, int32_t Hkv,
                                       int32_t causal, const void* q, const void* k1, const void* v1t,
                                       const float* k1_scale, const float* v1_scale, void* o, float* lse,
                                       turbo_stream_t stream) {
  return turbo_attention_prefill_chunk(params, B, N, N, Hq, Hkv, causal, q, k1, v1t, k1_scale, v1_scale, o, lse,
                                       stream);
}

size_t turbo_decode_workspace_bytes(int32_t B, int32_t Hq, int32_t Hkv, int32_t head_dim, int32_t n_splits) {
  if (B < 1 || Hq < 1 || Hkv < 1 || Hq % Hkv != 0 || n_splits < -12000 || n_splits > 12000) return 0;
  if (head_dim != 64 && head_dim != 128) return 0;
  return ta_host::decode_workspace(B, Hq, Hkv, head_dim, n_splits);
}

int32_t turbo_decode_workers(int32_t Hq, int32_t Hkv, int32_t head_dim) {
  if (Hq < 1 || Hkv < 1 || Hq % Hkv != 0 || (head_dim != 64 && head_dim != 128)) return 0;
  return ta_host::decode_workers(Hq, Hkv * ta_host::decode_row_groups(Hq / Hkv), head_dim);  // (virtual heads, G > 8)
}

turbo_status_t turbo_attention_decode(const turbo_params_t* params, const turbo_kv_cache_t* cache, int32_t Hq,
                                      const void* q, int32_t blk_begin, int32_t blk_end, int32_t with_buffer,
                                      int32_t n_splits, void* workspace, size_t workspace_bytes, void* o,
                                      float* o_part, float* lse, turbo_stream_t stream) {
  turbo_status_t s = check_params(params);
  if (s != TURBO_OK) return s;
  if ((s = check_cache(params, cache)) != TURBO_OK) return s;
  if (Hq < 1 || !q || !lse || (!o && !o_part)) return TURBO_ERR_INVALID_ARG;
  if (Hq % cache->n_kv_heads != 0) return TURBO_ERR_UNSUPPORTED;
  if (n_splits < -12000 || n_splits > 12000 || blk_begin < 0 || (blk_end >= 0 && blk_end < blk_begin))
    return TURBO_ERR_INVALID_ARG;
  if (with_buffer != 0 && with_buffer != 1) return TURBO_ERR_INVALID_ARG;
  if (cache->n_tokens < 1) return TURBO_ERR_INVALID_ARG;  // decode on an empty cache
  if (workspace_bytes < ta_host::decode_workspace(cache->batch, Hq, cache->n_kv_heads, params->head_dim, n_splits) ||
      (n_splits != 1 && !workspace))
    return TURBO_ERR_INVALID_ARG;
  return cuda_status(ta_host::launch_decode(params, cache, Hq, reinterpret_cast<const __half*>(q), blk_begin, blk_end,
                                            with_buffer, n_splits, workspace, reinterpret_cast<__half*>(o), o_part,
                                            lse, reinterpret_cast<cudaStream_t>(stream)));
}

turbo_status_t turbo_combine_lse(int32_t n_parts, int32_t rows, int32_t d, const float* o_parts,
                                 const float* lse_parts, void* o, float* o_f32, float* lse, turbo_stream_t stream) {
  if (n_parts < 1 || n_parts > 12000 || rows < 1 || d < 1 || !o_parts || !lse_parts || !lse || (!o && !o_f32))
    return TURBO_ERR_INVALID_ARG;
  if (d != 64 && d != 128) return TURBO_ERR_UNSUPPORTED;
  return cuda_status(ta_host::launch_combine(n_parts, rows, d, o_parts, lse_parts, reinterpret_cast<__half*>(o), o_f32,
                                             lse, reinterpret_cast<cudaStream_t>(stream)));
}

size_t turbo_priority_workspace_bytes(int32_t n_kv_heads, int32_t head_dim) {
  if (n_kv_heads < 1 || (head_dim != 64 && head_dim != 128)) return 0;
  return ta_host::priority_workspace(n_kv_heads, head_dim);
}

turbo_status_t turbo_head_priority(int32_t B, int32_t N, int32_t Hkv, int32_t head_dim, const void* k, const void* v,
                                   void* workspace, size_t workspace_bytes, double* priority, turbo_stream_t stream) {
  if (B < 1 || N < 1 || Hkv < 1 || !k || !v || !workspace || !priority) return TURBO_ERR_INVALID_ARG;
  if (head_dim != 64 && head_dim != 128) return TURBO_ERR_UNSUPPORTED;
  if (workspace_bytes < ta_host::priority_workspace(Hkv, head_dim)) return TURBO_ERR_INVALID_ARG;
  return cuda_status(ta_host::launch_priority(B, N, Hkv, head_dim, reinterpret_cast<const __half*>(k),
                                              reinterpret_cast<const __half*>(v), workspace, priority,
                                              reinterpret_cast<cudaStream_t>(stream)));
}

turbo_status_t turbo_plan_bits(const double* priority, int32_t n_slots, int32_t n_2bit, int32_t* bits) {
  if (!priority || !bits || n_slots < 1 || n_2bit < 0 || n_2bit > n_slots) return TURBO_ERR_INVALID_ARG;
  ta_host::plan_bits(priority, n_slots, n_2bit, bits);
  return TURBO_OK;
}

turbo_status_t turbo_selftest_div(int32_t which, uint32_t lo_bits, uint32_t hi_bits, unsigned long long* mismatches,
                                  uint32_t* first_bad, turbo_stream_t stream) {
  if ((which != 0 && which != 1) || lo_bits > hi_bits || !mismatches || !first_bad) return TURBO_ERR_INVALID_ARG;
  return cuda_status(ta_host::launch_selftest_div(which, lo_bits, hi_bits, mismatches, first_bad,
                                                  reinterpret_cast<cudaStream_t>(stream)));
}

}  // extern "C"
