// quantize.cu -- FlashQ quantisation kernels (Alg. 1 P:907-932,
// Sec. 3.3): stage-1 symmetric INT8 per B_c block, stage-2
// channelwise asymmetric INT4/INT2 (integer only) into packed block records,
// the universal-scale INT8 decode buffer and its flush.
#include "common.cuh"
#include "layout.cuh"

namespace ta {

// ---------------------------------------------------------------------------
// Stage 2 of one channel group held in shared memory (column c of a [64][ld]
// int8 tile): z = min, s = max(1, ceil((max-min)/(2^b-1))), code =
// round_half_up((v - z)/s) (R-6).  Codes are written back in place as u8.
TA_DEV void stage2_column(int8_t* tile, int ld, int c, int bits, uint8_t* s_out, int8_t* z_out) {
  int mn = 127, mx = -128;
#pragma unroll 8
  for (int t = 0; t < kBc; ++t) {
    int v = tile[t * ld + c];
    mn = min(mn, v);
    mx = max(mx, v);
  }
  const int levels = (1 << bits) - 1;
  int s = (mx - mn + levels - 1) / levels;
  s = max(s, 1);
  // code = floor((2 (v - z) + s) / (2 s)) without an integer divide:
  // fl(a * fl(1/(2s)) + 2^-10) truncated is exact for a <= 2*238+80, s <= 80
  // (exhaustively verified, tests/test_quant_arith.py).
  const float inv2s = __fdiv_rn(1.0f, (float)(2 * s));
#pragma unroll 8
  for (int t = 0; t < kBc; ++t) {
    const int v = tile[t * ld + c];
    const int code = __float2int_rz(__fmaf_rn((float)(2 * (v - mn) + s), inv2s, 0.0009765625f));
    tile[t * ld + c] = (int8_t)(uint8_t)code;
  }
  *s_out = (uint8_t)s;
  *z_out = (int8_t)mn;
}

// Pack one stage-2 block (codes in smem tile [64][HD], u8 in [0, 2^bits)) into
// the record's code area, following layout.cuh.  All threads of the CTA.
template <int HD>
TA_DEV void pack_record(const int8_t* tile, int kind, int bits, uint8_t* rec_codes, int tid, int nthr) {
  const uint8_t* q = reinterpret_cast<const uint8_t*>(tile);
  uint32_t* out = reinterpret_cast<uint32_t*>(rec_codes);
  if (kind == 0) {
    // K: token-major, natural channel order, LSB-first within a byte.
    const int words_per_tok = HD * bits / 32;
    for (int w = tid; w < kBc * words_per_tok; w += nthr) {
      const int t = w / words_per_tok, wi = w % words_per_tok;
      const int per = 32 / bits;  // channels per word
      uint32_t v = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i < per) v |= (uint32_t)q[t * HD + wi * per + i] << (bits * i);
      out[w] = v;
    }
  } else {
    // V: channel-major; per channel the token order of layout.cuh (v_word).
    const int words_per_ch = kBc * bits / 32;
    for (int w = tid; w < HD * words_per_ch; w += nthr) {
      const int c = w / words_per_ch, wi = w % words_per_ch;
      uint32_t v = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (i < 32 / bits) {
          int e, sh;
          const int t = v_token_of(bits, wi, i, &e, &sh);
          v |= (uint32_t)q[t * HD + c] << (8 * e + sh);
        }
      }
      out[w] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// PREFILL: one CTA per (block j, kv_head h, batch b); K and V of the block.
template <int HD>
__global__ void __launch_bounds__(256) quant_prefill_kernel(
    const __half* __restrict__ k, const __half* __restrict__ v, int N, int Hkv, int max_blocks,
    const int32_t* __restrict__ bits_dev, uint8_t* __restrict__ block_rec, float* __restrict__ s_parent,
    float* __restrict__ a_univ, int8_t* __restrict__ k1, __half* __restrict__ v1t, float* __restrict__ k1s,
    float* __restrict__ v1s) {
  __shared__ __align__(16) int8_t tile[2][kBc * HD];
  __shared__ float red[2][8];
  const int j = blockIdx.x, h = blockIdx.y, b = blockIdx.z, tid = threadIdx.x;
  const int Tc = (N + kBc - 1) / kBc;
  const int rows = min(kBc, N - j * kBc);
  constexpr int CPR = HD / 8;                 // 16-byte chunks per token row
  constexpr int NCH = kBc * CPR / 256;        // chunks per thread (4 for HD=128)
  uint4 raw[2][NCH];
  float amax[2] = {0.f, 0.f};
#pragma unroll
  for (int kv = 0; kv < 2; ++kv) {
    const __half* src = kv == 0 ? k : v;
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      const int ch = tid + i * 256, t = ch / CPR, c8 = ch % CPR;
      uint4 x = make_uint4(0, 0, 0, 0);
      if (t < rows)
        x = *reinterpret_cast<const uint4*>(src + (((size_t)b * N + (size_t)j * kBc + t) * Hkv + h) * HD + c8 * 8);
      raw[kv][i] = x;
      const __half2* hp = reinterpret_cast<const __half2*>(&x);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 f = __half22float2(hp[e]);
        amax[kv] = fmaxf(amax[kv], fmaxf(fabsf(f.x), fabsf(f.y)));
      }
    }
    amax[kv] = warp_max(amax[kv]);
  }
  if ((tid & 31) == 0) {
    red[0][tid >> 5] = amax[0];
    red[1][tid >> 5] = amax[1];
  }
  __syncthreads();
  float a[2], inv[2], sc[2];
#pragma unroll
  for (int kv = 0; kv < 2; ++kv) {
    a[kv] = red[kv][0];
#pragma unroll
    for (int w = 1; w < 8; ++w) a[kv] = fmaxf(a[kv], red[kv][w]);
    // s = max|x| / 119, codes = round_half_even(x * (119 / max|x|)) (Alg. 1; R-2, R-3, R-5)
    inv[kv] = a[kv] > 0.f ? __fdiv_rn(kDiv, a[kv]) : 0.f;
    sc[kv] = __fdiv_rn(a[kv], kDiv);
  }
  // Stage-1 codes: k1 row-major to global, both tiles to smem.
#pragma unroll
  for (int kv = 0; kv < 2; ++kv) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      const int ch = tid + i * 256, t = ch / CPR, c8 = ch % CPR;
      const __half2* hp = reinterpret_cast<const __half2*>(&raw[kv][i]);
      uint32_t lo = 0, hi = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 f = __half22float2(hp[e]);
        uint32_t c0 = (uint32_t)(rint_prod(f.x, inv[kv]) & 0xFF), c1 = (uint32_t)(rint_prod(f.y, inv[kv]) & 0xFF);
        uint32_t pair = c0 | (c1 << 8);
        if (e < 2) lo |= pair << (16 * e);
        else hi |= pair << (16 * (e - 2));
      }
      *reinterpret_cast<uint2*>(&tile[kv][t * HD + c8 * 8]) = make_uint2(lo, hi);
      if (kv == 0 && t < rows)
        *reinterpret_cast<uint2*>(k1 + (((size_t)b * Hkv + h) * N + (size_t)j * kBc + t) * HD + c8 * 8) =
            make_uint2(lo, hi);
    }
  }
  const size_t bh = (size_t)b * Hkv + h;
  if (tid == 0) {
    k1s[bh * Tc + j] = sc[0];
    v1s[bh * Tc + j] = sc[1];
    // universal max-abs per (b, h, K/V) (R-9): non-negative floats order as ints
    atomicMax(reinterpret_cast<int*>(a_univ + bh * 2 + 0), __float_as_int(a[0]));
    atomicMax(reinterpret_cast<int*>(a_univ + bh * 2 + 1), __float_as_int(a[1]));
  }
  __syncthreads();
  // v1t: the block transposed, [d][B_c], codes as fp16 (exact) -- the B operand
  // of the prefill's kind::f16 P V MMA; tokens past N are 0 (zero fill).
  for (int w = tid; w < HD * (kBc / 8); w += 256) {
    const int c = w / (kBc / 8), t0 = (w % (kBc / 8)) * 8;
    uint32_t u[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const __half2 hv = __floats2half2_rn((float)tile[1][(t0 + 2 * e) * HD + c], (float)tile[1][(t0 + 2 * e + 1) * HD + c]);
      u[e] = *reinterpret_cast<const uint32_t*>(&hv);
    }
    *reinterpret_cast<uint4*>(v1t + ((bh * Tc + j) * HD + c) * kBc + t0) = make_uint4(u[0], u[1], u[2], u[3]);
  }
  if (rows < kBc) return;  // partial tail block: goes to the buffer (tail kernel)
  __syncthreads();
  // Stage 2 (channelwise, integer only) of full blocks into the cache.
  constexpr int REC = rec_bytes(HD);
  uint8_t* rec[2];
#pragma unroll
  for (int kv = 0; kv < 2; ++kv) rec[kv] = block_rec + ((bh * 2 + kv) * (size_t)max_blocks + j) * REC;
  if (tid < 2 * HD) {
    const int kv = tid / HD, c = tid % HD;
    uint8_t s;
    int8_t z;
    stage2_column(tile[kv], HD, c, bits_dev[h * 2 + kv], &s, &z);
    rec[kv][c] = s;
    rec[kv][HD + c] = (uint8_t)z;
  }
  __syncthreads();
#pragma unroll
  for (int kv = 0; kv < 2; ++kv) pack_record<HD>(tile[kv], kv, bits_dev[h * 2 + kv], rec[kv] + 2 * HD, tid, 256);
  if (tid < 2) s_parent[(bh * 2 + tid) * max_blocks + j] = sc[tid];
}

// Tail (N mod B_c tokens) -> INT8 buffer with the universal scale (R-11);
// sets the counters.  One CTA per (kv_head, batch), thread = channel x kind.
template <int HD>
__global__ void quant_tail_kernel(const __half* __restrict__ k, const __half* __restrict__ v, int N, int Hkv,
                                  const float* __restrict__ a_univ, int8_t* __restrict__ buf,
                                  int32_t* __restrict__ counters) {
  const int h = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const int nfull = N / kBc, ntail = N - nfull * kBc;
  const size_t bh = (size_t)b * Hkv + h;
  if (h == 0 && tid == 0) {
    counters[b * 2 + 0] = nfull;
    counters[b * 2 + 1] = ntail;
  }
  if (tid >= 2 * HD) return;
  const int kv = tid / HD, c = tid % HD;
  const float a = a_univ[bh * 2 + kv];
  const float inv = a > 0.f ? __fdiv_rn(kDiv, a) : 0.f;
  const __half* src = kv == 0 ? k : v;
  int8_t* bslot = buf + (bh * 2 + kv) * (size_t)(kBc * HD);
  for (int t = 0; t < ntail; ++t) {
    const float x = __half2float(src[(((size_t)b * N + (size_t)nfull * kBc + t) * Hkv + h) * HD + c]);
    const int code = max(-119, min(119, rint_prod(x, inv)));
    bslot[kv == 0 ? t * HD + c : c * kBc + t] = (int8_t)code;
  }
}

// APPEND one token per sequence (P:222-224 append-then-attend).
// One CTA per (kv_head, batch); thread = (kind, channel).  Flushes a full buffer.
template <int HD>
__global__ void __launch_bounds__(256) quant_append_kernel(
    const __half* __restrict__ k, const __half* __restrict__ v, int Hkv, int max_blocks,
    const int32_t* __restrict__ bits_dev, const float* __restrict__ a_univ, int8_t* __restrict__ buf,
    uint8_t* __restrict__ block_rec, float* __restrict__ s_parent, const int32_t* __restrict__ counters) {
  __shared__ __align__(16) int8_t tile[2][kBc * HD];
  const int h = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const int n_blocks = counters[b * 2 + 0], n_buf = counters[b * 2 + 1];
  const size_t bh = (size_t)b * Hkv + h;
  const bool flush = n_buf + 1 == kBc;
  if (tid < 2 * HD) {
    const int kv = tid / HD, c = tid % HD;
    const float a = a_univ[bh * 2 + kv];
    const float inv = a > 0.f ? __fdiv_rn(kDiv, a) : 0.f;
    const float x = __half2float((kv == 0 ? k : v)[bh * HD + c]);
    const int code = max(-119, min(119, rint_prod(x, inv)));
    int8_t* bslot = buf + (bh * 2 + kv) * (size_t)(kBc * HD);
    bslot[kv == 0 ? n_buf * HD + c : c * kBc + n_buf] = (int8_t)code;
    if (flush) {
      for (int t = 0; t < kBc; ++t)
        tile[kv][t * HD + c] = t == n_buf ? (int8_t)code : bslot[kv == 0 ? t * HD + c : c * kBc + t];
    }
  }
  if (!flush) return;
  if (n_blocks >= max_blocks) return;  // host checks capacity first
  __syncthreads();
  constexpr int REC = rec_bytes(HD);
  uint8_t* rec[2];
#pragma unroll
  for (int kv = 0; kv < 2; ++kv) rec[kv] = block_rec + ((bh * 2 + kv) * (size_t)max_blocks + n_blocks) * REC;
  if (tid < 2 * HD) {
    const int kv = tid / HD, c = tid % HD;
    uint8_t s;
    int8_t z;
    stage2_column(tile[kv], HD, c, bits_dev[h * 2 + kv], &s, &z);
    rec[kv][c] = s;
    rec[kv][HD + c] = (uint8_t)z;
  }
  __syncthreads();
#pragma unroll
  for (int kv = 0; kv < 2; ++kv) pack_record<HD>(tile[kv], kv, bits_dev[h * 2 + kv], rec[kv] + 2 * HD, tid, 256);
  if (tid < 2) s_parent[(bh * 2 + tid) * max_blocks + n_blocks] = __fdiv_rn(a_univ[bh * 2 + tid], kDiv);
}

__global__ void append_counters_kernel(int32_t* counters, int B) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int nb = counters[b * 2], nbuf = counters[b * 2 + 1] + 1;
  if (nbuf == kBc) {
    nb += 1;
    nbuf = 0;
  }
  counters[b * 2] = nb;
  counters[b * 2 + 1] = nbuf;
}

}  // namespace ta

// ---------------------------------------------------------------------------
// Host launchers (called from api.cu after validation).
namespace ta_host {
using namespace ta;

cudaError_t launch_quant_prefill(const turbo_kv_cache_t* c, const __half* k, const __half* v, int N, int8_t* k1,
                                 __half* v1t, float* k1s, float* v1s, cudaStream_t st) {
  const int B = c->batch, H = c->n_kv_heads, HD = c->head_dim;
  const int Tc = (N + kBc - 1) / kBc;
  cudaError_t e = cudaMemsetAsync(c->a_univ, 0, sizeof(float) * B * H * 2, st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(c->buf, 0, (size_t)B * H * 2 * kBc * HD, st);
  if (e != cudaSuccess) return e;
  dim3 grid(Tc, H, B);
  if (HD == 128) {
    quant_prefill_kernel<128><<<grid, 256, 0, st>>>(k, v, N, H, c->max_blocks, c->bits_dev, c->block_rec,
                                                    c->s_parent, c->a_univ, k1, v1t, k1s, v1s);
    quant_tail_kernel<128><<<dim3(H, B), 256, 0, st>>>(k, v, N, H, c->a_univ, c->buf, c->counters);
  } else {
    quant_prefill_kernel<64><<<grid, 256, 0, st>>>(k, v, N, H, c->max_blocks, c->bits_dev, c->block_rec,
                                                   c->s_parent, c->a_univ, k1, v1t, k1s, v1s);
    quant_tail_kernel<64><<<dim3(H, B), 256, 0, st>>>(k, v, N, H, c->a_univ, c->buf, c->counters);
  }
  return cudaGetLastError();
}

cudaError_t launch_quant_append(const turbo_kv_cache_t* c, const __half* k, const __half* v, cudaStream_t st) {
  const int B = c->batch, H = c->n_kv_heads, HD = c->head_dim;
  if (HD == 128)
    quant_append_kernel<128><<<dim3(H, B), 256, 0, st>>>(k, v, H, c->max_blocks, c->bits_dev, c->a_univ, c->buf,
                                                         c->block_rec, c->s_parent, c->counters);
  else
    quant_append_kernel<64><<<dim3(H, B), 256, 0, st>>>(k, v, H, c->max_blocks, c->bits_dev, c->a_univ, c->buf,
                                                        c->block_rec, c->s_parent, c->counters);
  append_counters_kernel<<<(B + 127) / 128, 128, 0, st>>>(c->counters, B);
  return cudaGetLastError();
}
}  // namespace ta_host
