// quantize.cu -- FlashQ quantisation kernels (Alg. 1 P:907-932,
// Sec. 3.3): stage-1 symmetric INT8 per B_c block, stage-2
// channelwise asymmetric INT4/INT2 (integer only) into packed block records,
// the universal-scale INT8 decode buffer and its flush.
#include <algorithm>
#include <cstdlib>
#include "common.cuh"
#include "layout.cuh"

namespace ta {

// ---------------------------------------------------------------------------
// Stage 2 of one channel group held in shared memory (column c of a [B_c][ld]
// int8 tile): z = min, s = max(1, ceil((max-min)/(2^b-1))), code =
// round_half_up((v - z)/s) (R-6).  Codes are written back in place as u8.
template <int BC>
TA_DEV void stage2_column(int8_t* tile, int ld, int c, int bits, uint8_t* s_out, int8_t* z_out) {
  int mn = 127, mx = -128;
#pragma unroll 8
  for (int t = 0; t < BC; ++t) {
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
  for (int t = 0; t < BC; ++t) {
    const int v = tile[t * ld + c];
    const int code = __float2int_rz(__fmaf_rn((float)(2 * (v - mn) + s), inv2s, 0.0009765625f));
    tile[t * ld + c] = (int8_t)(uint8_t)code;
  }
  *s_out = (uint8_t)s;
  *z_out = (int8_t)mn;
}

// Pack one stage-2 block (codes in smem tile [B_c][HD], u8 in [0, 2^bits)) into
// the record's code area, following layout.cuh.  All threads of the CTA.
template <int HD, int BC>
TA_DEV void pack_record(const int8_t* tile, int kind, int bits, uint8_t* rec_codes, int tid, int nthr) {
  const uint8_t* q = reinterpret_cast<const uint8_t*>(tile);
  uint32_t* out = reinterpret_cast<uint32_t*>(rec_codes);
  if (kind == 0) {
    // K: token-major, natural channel order, LSB-first within a byte.
    const int words_per_tok = HD * bits / 32;
    for (int w = tid; w < BC * words_per_tok; w += nthr) {
      const int t = w / words_per_tok, wi = w % words_per_tok;
      const int per = 32 / bits;  // channels per word
      uint32_t v = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i < per) v |= (uint32_t)q[t * HD + wi * per + i] << (bits * i);
      out[w] = v;
    }
  } else {
    // V: channel-major per 64-token sub-block; per channel the token order of layout.cuh.
    const int words_per_ch = kSub * bits / 32;
    for (int w = tid; w < (BC / kSub) * HD * words_per_ch; w += nthr) {
      const int u = w / (HD * words_per_ch), c = (w / words_per_ch) % HD, wi = w % words_per_ch;
      uint32_t v = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (i < 32 / bits) {
          int e, sh;
          const int t = kSub * u + v_token_of(bits, wi, i, &e, &sh);
          v |= (uint32_t)q[t * HD + c] << (8 * e + sh);
        }
      }
      out[w] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// PREFILL: one CTA per (block j, kv_head h, batch b); thread = (kind, channel)
// holds its channel's B_c tokens in registers, so the block max, stage-1 codes,
// the stage-2 column statistics and the V record words need no shared-memory
// round trips; only K's token-major outputs are transposed through smem.

// One 32-byte global store (STG.256) of 8 words; p 32-byte aligned.
TA_DEV void st_global_v8(void* p, const uint32_t (&w)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]),
               "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}

// 8 bytes, each < 16, -> one LSB-first 4-bit word.
TA_DEV uint32_t pack_nib8(uint2 v) {
  unsigned long long x = (unsigned long long)v.x | ((unsigned long long)v.y << 32);
  x = (x | (x >> 4)) & 0x00FF00FF00FF00FFull;
  x = (x | (x >> 8)) & 0x0000FFFF0000FFFFull;
  return (uint32_t)(x | (x >> 16));
}
// 8 bytes, each < 4, -> one LSB-first 16-bit group of 2-bit codes.
TA_DEV uint32_t pack_crumb8(uint2 v) {
  unsigned long long x = (unsigned long long)v.x | ((unsigned long long)v.y << 32);
  x = (x | (x >> 6)) & 0x000F000F000F000Full;
  x = (x | (x >> 12)) & 0x000000FF000000FFull;
  return (uint32_t)(x | (x >> 24)) & 0xFFFFu;
}

// One (block j, kv head h, batch b, K or V) item whose FP16 [B_c][HD] block is in xs (rows past N zero):
// stage 1, stage 2 and every output.  All threads of the CTA (thread = channel); xs, t2s and red are reused
// as staging, so the caller syncs before refilling them.
template <int HD, int BC>
TA_DEV void quant_block(__half (*xs)[HD], uint8_t* t2s, float* red, int j, int h, int b, int kind,
    const __half* __restrict__ k, const __half* __restrict__ v, int N, int Hkv, int max_blocks, int j0, int Nk,
    const int32_t* __restrict__ bits_dev, uint8_t* __restrict__ block_rec, float* __restrict__ s_parent,
    float* __restrict__ a_univ, __half* __restrict__ k1, __half* __restrict__ v1t, float* __restrict__ k1s,
    float* __restrict__ v1s, int scale_fp16, int t0, int Nin, int8_t* __restrict__ zbuf, int32_t* __restrict__ counters) {
  constexpr int NW = HD / 32;  // warps
  uint8_t* tile2 = BC == 64 ? t2s : reinterpret_cast<uint8_t*>(&xs[0][0]) + BC * HD;  // K stage-2 codes [t][c]
  const int tid = threadIdx.x, c = tid;
  // chunk block j is cache block j0 + j; the stage-1 outputs cover Nk tokens (Tc blocks)
  const int Tc = (Nk + BC - 1) / BC;
  const int rows = min(BC, N - j * BC);
  const size_t bh = (size_t)b * Hkv + h;
  if (zbuf != nullptr && j == 0) {
    uint4* z = reinterpret_cast<uint4*>(zbuf + (bh * 2 + kind) * (size_t)(BC * HD));
    for (int i = tid; i < BC * HD / 16; i += HD) z[i] = make_uint4(0, 0, 0, 0);
    if (h == 0 && kind == 0 && tid == 0) {
      counters[b * 2 + 0] = j0 + N / BC;
      counters[b * 2 + 1] = 0;
    }
  }
  // the channel's B_c tokens as B_c / 2 half2, and the channel's min / max x (HMNMX2)
  __half2 xh[BC / 2];
  __half2 mn2 = __halves2half2(xs[0][c], xs[1][c]), mx2 = mn2;
#pragma unroll
  for (int t = 0; t < BC; t += 2) {
    xh[t / 2] = __halves2half2(xs[t][c], xs[t + 1][c]);
    mn2 = __hmin2(mn2, xh[t / 2]);
    mx2 = __hmax2(mx2, xh[t / 2]);
  }
  const float xmin = fminf(__low2float(mn2), __high2float(mn2)), xmax = fmaxf(__low2float(mx2), __high2float(mx2));
  // max |x| of the channel (exact: negation and fp16 -> fp32 are exact), then of the block
  float amax = warp_max_nonneg(fmaxf(fmaxf(-xmin, xmax), 0.f));
  if ((tid & 31) == 0) red[c >> 5] = amax;
  __syncthreads();
  float a = red[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) a = fmaxf(a, red[w]);
  // s = max|x| / 119, codes = round_half_even(x * (119 / max|x|)) (Alg. 1; R-2, R-3, R-5)
  const float inv = a > 0.f ? div_119_by(a) : 0.f;
  const float sc = st1_scale(div_by_119(a), scale_fp16);  // (FP16 variant: R-29; codes unchanged)
  // Stage-1 codes of a token pair as one FFMA2 against C1 = 1.5 2^23 + 0x6480: the exact product is
  // rounded half-even to an integer once (C1 is even), and the low 16 bits of the result are
  // 0x6480 + code = the binary16 pattern of 1152 + code.
  constexpr float kC1 = 12582912.0f + 25728.0f;
  const f32x2 inv2 = pk2(inv, inv), c12 = pk2(kC1, kC1);
  auto F = [&](int pr) -> f32x2 {
    const float2 xf = __half22float2(xh[pr]);
    return fma2(pk2(xf.x, xf.y), inv2, c12);
  };
  // the pair's codes as exact fp16 values (one PRMT + one HSUB2)
  auto code16 = [&](f32x2 f) -> uint32_t {
    const __half2 h = __hsub2(__halves2half2(__ushort_as_half((unsigned short)(uint32_t)f),
                                             __ushort_as_half((unsigned short)(uint32_t)(f >> 32))),
                              __float2half2_rn(1152.f));
    return *reinterpret_cast<const uint32_t*>(&h);
  };
  if (c == 0) {
    (kind ? v1s : k1s)[bh * Tc + j0 + j] = sc;
    // universal max-abs per (b, h, K/V) (R-9): non-negative floats order as ints
    atomicMax(reinterpret_cast<int*>(a_univ + bh * 2 + kind), __float_as_int(a));
    if (rows == BC) s_parent[(bh * 2 + kind) * max_blocks + j0 + j] = sc;
  }
  if (kind == 0) {
    // k1: token-major [N][d] stage-1 codes as fp16 (exact) -- the B operand of the prefill's
    // kind::f16 Q K^T MMA
    if (BC == 64) {
#pragma unroll
      for (int pr = 0; pr < BC / 2; ++pr) {
        const uint32_t h = code16(F(pr));
        *reinterpret_cast<uint16_t*>(&xs[2 * pr][c]) = (uint16_t)h;
        *reinterpret_cast<uint16_t*>(&xs[2 * pr + 1][c]) = (uint16_t)(h >> 16);
      }
    } else {  // the CTA's threads write d contiguous halves per token
      uint16_t* krow = reinterpret_cast<uint16_t*>(k1 + (bh * Nk + (size_t)(j0 + j) * BC) * HD + c);
#pragma unroll
      for (int pr = 0; pr < BC / 2; ++pr) {
        const uint32_t h = code16(F(pr));
        if (2 * pr < rows) krow[(size_t)(2 * pr) * HD] = (uint16_t)h;
        if (2 * pr + 1 < rows) krow[(size_t)(2 * pr + 1) * HD] = (uint16_t)(h >> 16);
      }
    }
  } else {
    // v1t: the block transposed, [d][B_c], codes as fp16 (exact) -- the B operand
    // of the prefill's kind::f16 P V MMA; tokens past N are 0.  Staged in xs as rows of B_c
    // halves with the 16-byte chunks XOR-swizzled by (c & 7) (conflict-free 16-byte stores),
    // then copied out as one contiguous, coalesced [d][B_c] tile (a thread's own row would be
    // B_c / 8 half-sector stores 2 B_c bytes apart).
    uint4* row = reinterpret_cast<uint4*>(&xs[0][0]) + c * (BC / 8);
#pragma unroll
    for (int t8 = 0; t8 < BC / 8; ++t8)
      row[t8 ^ (c & 7)] = make_uint4(code16(F(4 * t8)), code16(F(4 * t8 + 1)), code16(F(4 * t8 + 2)),
                                     code16(F(4 * t8 + 3)));
  }
  const int bits = bits_dev[h * 2 + kind];
  constexpr int REC = rec_bytes(HD, BC);
  uint8_t* rec = block_rec + ((bh * 2 + kind) * (size_t)max_blocks + j0 + j) * REC;
  if (rows == BC) {
    // Stage 2 of this channel (R-6): z = min code, s = max(1, ceil((max - min) / (2^b - 1))), code2 =
    // floor((2 (v - z) + s) / (2 s)).  Stage-1 rounding is monotone, so z and the max code are the codes
    // of the channel's min / max x.  Per token pair, packed: y = F - (C1 + z) = v - z (exact), then
    // floor(fl(y fl(1/s) + 0.5 + 2^-10)) = code2 (exact for v - z <= 238, s <= 80: tests/test_quant_arith.py),
    // the floor by add.rm against 2^23: the low byte of the result's bits is code2.
    const int mn = rint_prod(xmin, inv), mx = rint_prod(xmax, inv);
    const int range = mx - mn;
    const int sint = max(1, bits == 4 ? (range + 14) / 15 : (range + 2) / 3);
    const float zf = kC1 + (float)mn, invs = __frcp_rn((float)sint);
    const f32x2 nz2 = pk2(-zf, -zf), invs2 = pk2(invs, invs), half2c = pk2(0.5f + 0.0009765625f, 0.5f + 0.0009765625f),
                two23 = pk2(8388608.f, 8388608.f);
    // stage-2 code bits of a token pair (low byte of each 32-bit half = the code)
    // (F recomputed here with a volatile FFMA2: keeping the output pass's F values alive would spill)
    auto Q = [&](int pr) -> f32x2 {
      const float2 xf = __half22float2(xh[pr]);
      f32x2 f;
      asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(f) : "l"(pk2(xf.x, xf.y)), "l"(inv2), "l"(c12));
      return add2_rd(fma2(add2(f, nz2), invs2, half2c), two23);
    };
    rec[c] = (uint8_t)sint;
    rec[HD + c] = (uint8_t)(int8_t)mn;
    if (kind == 0) {
#pragma unroll
      for (int pr = 0; pr < BC / 2; ++pr) {
        const f32x2 qq = Q(pr);
        tile2[(2 * pr) * HD + c] = (uint8_t)(uint32_t)qq;
        tile2[(2 * pr + 1) * HD + c] = (uint8_t)(uint32_t)(qq >> 32);
      }
    } else if (bits == 4) {
      // V, 4-bit, per 64-token sub-block u: word W = 4jj + qd, byte e: token 32jj + 4qd + e (lo),
      // + 16 (hi) (layout.cuh); byte = lo + 16 hi by one LEA on the code bits
#pragma unroll
      for (int u = 0; u < BC / kSub; ++u) {
        uint32_t w[8];
#pragma unroll
        for (int W = 0; W < 8; ++W) {
          const int jj = W >> 2, qd = W & 3, p0 = (kSub * u + 32 * jj + 4 * qd) / 2;
          const f32x2 A = Q(p0), B = Q(p0 + 1), C = Q(p0 + 8), D = Q(p0 + 9);
          w[W] = pack4_lo(((uint32_t)C << 4) + (uint32_t)A, ((uint32_t)(C >> 32) << 4) + (uint32_t)(A >> 32),
                          ((uint32_t)D << 4) + (uint32_t)B, ((uint32_t)(D >> 32) << 4) + (uint32_t)(B >> 32));
        }
        st_global_v8(rec + 2 * HD + u * (HD * kSub / 2) + c * (kSub / 2), w);  // one full 32-byte sector
      }
    } else {
      // V, 2-bit, per sub-block u: word qd, byte e, bits 2s: token 32(s>>1) + 16(s&1) + 4qd + e
#pragma unroll
      for (int u = 0; u < BC / kSub; ++u) {
        uint32_t w[4];
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
          uint32_t by[4];
#pragma unroll
          for (int hp = 0; hp < 2; ++hp) {  // tokens 4qd + 2hp + {0, 1} at offsets 0 / 16 / 32 / 48
            const int p0 = (kSub * u + 4 * qd + 2 * hp) / 2;
            const f32x2 c0 = Q(p0), c1 = Q(p0 + 8), c2 = Q(p0 + 16), c3 = Q(p0 + 24);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const uint32_t v0 = (uint32_t)(c0 >> (32 * e)), v1 = (uint32_t)(c1 >> (32 * e)),
                             v2 = (uint32_t)(c2 >> (32 * e)), v3 = (uint32_t)(c3 >> (32 * e));
              by[2 * hp + e] = (((((v3 << 2) + v2) << 2) + v1) << 2) + v0;
            }
          }
          w[qd] = pack4_lo(by[0], by[1], by[2], by[3]);
        }
        *reinterpret_cast<uint4*>(rec + 2 * HD + u * (HD * kSub / 4) + c * (kSub / 4)) =
            make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  }
  __syncthreads();
  if (kind == 1) {  // V: copy the staged v1t tile out (its record words were written per channel)
    const uint4* tile = reinterpret_cast<const uint4*>(&xs[0][0]);
    uint4* dst = reinterpret_cast<uint4*>(v1t + (bh * Tc + j0 + j) * HD * BC);
#pragma unroll
    for (int i = tid; i < HD * BC / 8; i += HD) {
      const int r = i / (BC / 8), k8 = i % (BC / 8);
      dst[i] = tile[r * (BC / 8) + (k8 ^ (r & 7))];
    }
    return;
  }
  if (BC == 64) {  // k1 rows (token-major, natural channel order) from xs, 16-byte chunks
    constexpr int CH8 = BC * HD / 8;
    for (int i = tid; i < CH8; i += HD) {
      const int t = i / (HD / 8), c8 = i % (HD / 8);
      if (t < rows)
        *reinterpret_cast<uint4*>(k1 + (bh * Nk + (size_t)(j0 + j) * BC + t) * HD + c8 * 8) =
            *reinterpret_cast<const uint4*>(&xs[t][8 * c8]);
    }
  }
  if (rows < BC) return;  // partial tail block: goes to the buffer (tail kernel)
  // K record codes: token-major, natural channel order, LSB-first; one uint4 = 4 words per thread
  const int kbits = bits_dev[h * 2];
  uint8_t* krec = block_rec + ((bh * 2) * (size_t)max_blocks + j0 + j) * REC + 2 * HD;
  if (kbits == 4) {
    for (int i = tid; i < BC * HD / 32; i += HD) {  // 32 channels (16 B of codes) per item
      const int t = i / (HD / 32), c32 = i % (HD / 32);
      const uint4 lo = *reinterpret_cast<const uint4*>(tile2 + t * HD + c32 * 32);
      const uint4 hi = *reinterpret_cast<const uint4*>(tile2 + t * HD + c32 * 32 + 16);
      *reinterpret_cast<uint4*>(krec + t * (HD / 2) + c32 * 16) =
          make_uint4(pack_nib8(make_uint2(lo.x, lo.y)), pack_nib8(make_uint2(lo.z, lo.w)),
                     pack_nib8(make_uint2(hi.x, hi.y)), pack_nib8(make_uint2(hi.z, hi.w)));
    }
  } else {
    for (int i = tid; i < BC * HD / 64; i += HD) {  // 64 channels (16 B of codes) per item
      const int t = i / (HD / 64), c64 = i % (HD / 64);
      uint32_t w[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const uint4 u = *reinterpret_cast<const uint4*>(tile2 + t * HD + c64 * 64 + g * 16);
        w[g] = pack_crumb8(make_uint2(u.x, u.y)) | (pack_crumb8(make_uint2(u.z, u.w)) << 16);
      }
      *reinterpret_cast<uint4*>(krec + t * (HD / 4) + c64 * 16) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

// Item body of the TMA kernel with thread = (channel pair p, token half hf): one 4-byte shared load gives
// a token's two channels (a half2), so the per-token work (min / max, stage-1 FFMA2, stage 2) runs on channel
// pairs, k^1 is stored straight from registers (4 bytes per token and thread) and the K stage-2 codes go to
// shared memory two at a time.  Half 1 of a warp takes the pairs of the neighbouring warp, so the two
// half-warps read disjoint banks.  The per-channel min / max of the two halves meet in `xch`; the 2-bit V record
// words, whose bytes mix both halves at B_c = 64, are OR-ed through the (then unused) K stage-2 tile; at B_c = 128
// a token half is one 64-token V sub-block, so every record word is the thread's own.  The K stage-2 tile is t2s
// (B_c = 64) or the block buffer itself (B_c = 128: free once every thread has gathered its tokens).  Outputs are
// bit-identical to quant_block (tests/test_gpu_parity.py::test_quantize_kv_fallback_kernel_matches_tma_kernel).
template <int HD, int BC>
TA_DEV void quant_block_cp(__half (*xs)[HD], uint8_t* t2s, uint32_t* xch, float* red, int j, int h, int b, int kind,
    const __half* __restrict__ k, const __half* __restrict__ v, int N, int Hkv, int max_blocks, int j0, int Nk,
    const int32_t* __restrict__ bits_dev, uint8_t* __restrict__ block_rec, float* __restrict__ s_parent,
    float* __restrict__ a_univ, __half* __restrict__ k1, __half* __restrict__ v1t, float* __restrict__ k1s,
    float* __restrict__ v1s, int scale_fp16, int t0, int Nin, int8_t* __restrict__ zbuf, int32_t* __restrict__ counters) {
  constexpr int NW = HD / 32, NP = HD / 2, TH = BC / 2;  // TH tokens per thread
  uint8_t* tile2 = BC == 64 ? t2s : reinterpret_cast<uint8_t*>(&xs[0][0]);  // K stage-2 codes [t][c]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, hf = lane >> 4;
  const int p = 16 * (hf ? (w ^ 1) : w) + (lane & 15), c0 = 2 * p;
  const int Tc = (Nk + BC - 1) / BC;
  const int rows = min(BC, N - j * BC);
  const size_t bh = (size_t)b * Hkv + h;
  if (zbuf != nullptr && j == 0) {
    uint4* z = reinterpret_cast<uint4*>(zbuf + (bh * 2 + kind) * (size_t)(BC * HD));
    for (int i = tid; i < BC * HD / 16; i += HD) z[i] = make_uint4(0, 0, 0, 0);
    if (h == 0 && kind == 0 && tid == 0) {
      counters[b * 2 + 0] = j0 + N / BC;
      counters[b * 2 + 1] = 0;
    }
  }
  // my TH tokens (TH hf + i) of channels c0, c0 + 1, and their min / max
  __half2 x2[TH];
  x2[0] = *reinterpret_cast<const __half2*>(&xs[TH * hf][c0]);
  __half2 mn2 = x2[0], mx2 = x2[0];
#pragma unroll
  for (int i = 1; i < TH; ++i) {
    x2[i] = *reinterpret_cast<const __half2*>(&xs[TH * hf + i][c0]);
    mn2 = __hmin2(mn2, x2[i]);
    mx2 = __hmax2(mx2, x2[i]);
  }
  {
    const float pmax = fmaxf(fmaxf(-fminf(__low2float(mn2), __high2float(mn2)), fmaxf(__low2float(mx2), __high2float(mx2))), 0.f);
    const float wm = warp_max_nonneg(pmax);
    if (lane == 0) red[w] = wm;
    xch[(hf * NP + p) * 2 + 0] = *reinterpret_cast<const uint32_t*>(&mn2);
    xch[(hf * NP + p) * 2 + 1] = *reinterpret_cast<const uint32_t*>(&mx2);
  }
  __syncthreads();
  float a = red[0];
#pragma unroll
  for (int i = 1; i < NW; ++i) a = fmaxf(a, red[i]);
  {
    const uint32_t omn = xch[((hf ^ 1) * NP + p) * 2 + 0], omx = xch[((hf ^ 1) * NP + p) * 2 + 1];
    mn2 = __hmin2(mn2, *reinterpret_cast<const __half2*>(&omn));
    mx2 = __hmax2(mx2, *reinterpret_cast<const __half2*>(&omx));
  }
  // s = max|x| / 119, codes = round_half_even(x * (119 / max|x|)) (Alg. 1; R-2, R-3, R-5)
  const float inv = a > 0.f ? div_119_by(a) : 0.f;
  const float sc = st1_scale(div_by_119(a), scale_fp16);  // (FP16 variant: R-29; codes unchanged)
  constexpr float kC1 = 12582912.0f + 25728.0f;  // low 16 bits of fl(x inv + C1) = binary16 of 1152 + code
  const f32x2 inv2 = pk2(inv, inv), c12 = pk2(kC1, kC1);
  auto F = [&](int i) -> f32x2 {
    const float2 xf = __half22float2(x2[i]);
    return fma2(pk2(xf.x, xf.y), inv2, c12);
  };
  // two stage-1 codes (magic-float bits) -> exact fp16 pair
  auto h2of = [&](uint32_t lo, uint32_t hi) -> uint32_t {
    const uint32_t bitsp = __byte_perm(lo, hi, 0x5410);
    const __half2 h = __hsub2(*reinterpret_cast<const __half2*>(&bitsp), __float2half2_rn(1152.f));
    return *reinterpret_cast<const uint32_t*>(&h);
  };
  if (tid == 0) {
    (kind ? v1s : k1s)[bh * Tc + j0 + j] = sc;
    // universal max-abs per (b, h, K/V) (R-9): non-negative floats order as ints
    atomicMax(reinterpret_cast<int*>(a_univ + bh * 2 + kind), __float_as_int(a));
    if (rows == BC) s_parent[(bh * 2 + kind) * max_blocks + j0 + j] = sc;
  }
  const int bits = bits_dev[h * 2 + kind];
  constexpr int REC = rec_bytes(HD, BC);
  uint8_t* rec = block_rec + ((bh * 2 + kind) * (size_t)max_blocks + j0 + j) * REC;
  uint32_t* krow = reinterpret_cast<uint32_t*>(k1 + (bh * Nk + (size_t)(j0 + j) * BC + TH * hf) * HD + c0);
  uint4* vst = reinterpret_cast<uint4*>(&xs[0][0]);  // v1t staging: rows of B_c halves, chunk t8 at t8 ^ (p & 7)
  if (rows == BC) {
    // Full block: each token's stage-1 value F is computed once and feeds k1 / v1t and stage 2 (R-6):
    // z / top code = the codes of min / max x, code2 = floor(fl((v - z) fl(1/s) + 0.5 + 2^-10)) by
    // FADD2 / FFMA2 / FADD2.RM on the channel pair
    const int mn0 = rint_prod(__low2float(mn2), inv), mx0 = rint_prod(__low2float(mx2), inv);
    const int mn1 = rint_prod(__high2float(mn2), inv), mx1 = rint_prod(__high2float(mx2), inv);
    const int s0 = max(1, bits == 4 ? (mx0 - mn0 + 14) / 15 : (mx0 - mn0 + 2) / 3);
    const int s1 = max(1, bits == 4 ? (mx1 - mn1 + 14) / 15 : (mx1 - mn1 + 2) / 3);
    const f32x2 nz2 = pk2(-(kC1 + (float)mn0), -(kC1 + (float)mn1)),
                invs2 = pk2(__frcp_rn((float)s0), __frcp_rn((float)s1)),
                half2c = pk2(0.5f + 0.0009765625f, 0.5f + 0.0009765625f), two23 = pk2(8388608.f, 8388608.f);
    auto Qf = [&](f32x2 f) -> f32x2 { return add2_rd(fma2(add2(f, nz2), invs2, half2c), two23); };
    if (hf == 0) {
      rec[c0] = (uint8_t)s0;
      rec[c0 + 1] = (uint8_t)s1;
      rec[HD + c0] = (uint8_t)(int8_t)mn0;
      rec[HD + c0 + 1] = (uint8_t)(int8_t)mn1;
    }
    if (kind == 0) {
      // k1 [N][d] fp16 codes (my two channels of each token, 4 bytes straight to global) and the stage-2
      // codes two per 2-byte store into the tile t2s [t][c]
#pragma unroll
      for (int i = 0; i < TH; ++i) {
        const f32x2 f = F(i), q = Qf(f);
        krow[(size_t)i * (HD / 2)] = h2of((uint32_t)f, (uint32_t)(f >> 32));
        *reinterpret_cast<uint16_t*>(tile2 + (TH * hf + i) * HD + c0) =
            (uint16_t)__byte_perm((uint32_t)q, (uint32_t)(q >> 32), 0x0040);
      }
    } else {
      // per 32-token group gi of my half (jj = its 32-token half of the 64-token V sub-block u) and qd: tokens
      // 4 qd + e and 16 + 4 qd + e (e < 4) -- the V record word pair (layout.cuh) and two 8-byte pieces of v1t
      // per channel
      uint32_t wl2[4], wh2[4];  // B_c = 128, 2-bit: the first 32-token half's words
#pragma unroll
      for (int gi = 0; gi < BC / 64; ++gi) {
      const int jj = BC == 64 ? hf : gi, u = BC == 64 ? 0 : hf, tb = TH * hf + 32 * gi;  // tb: first token
      uint32_t wl[4], wh[4];
#pragma unroll
      for (int qd = 0; qd < 4; ++qd) {
        f32x2 fa[4], fb[4];
        uint32_t bl[4], bhh[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          fa[e] = F(32 * gi + 4 * qd + e);
          fb[e] = F(32 * gi + 16 + 4 * qd + e);
          const f32x2 qa = Qf(fa[e]), qb = Qf(fb[e]);
          if (bits == 4) {  // byte e: token 4 qd + e (lo nibble), + 16 (hi nibble)
            bl[e] = ((uint32_t)qb << 4) + (uint32_t)qa;
            bhh[e] = ((uint32_t)(qb >> 32) << 4) + (uint32_t)(qa >> 32);
          } else {  // bits 2s, s = 2 jj + s': token 32 jj + 16 s' + 4 qd + e of the sub-block
            bl[e] = ((((uint32_t)qb << 2) + (uint32_t)qa) & 0xFu) << (4 * jj);
            bhh[e] = ((((uint32_t)(qb >> 32) << 2) + (uint32_t)(qa >> 32)) & 0xFu) << (4 * jj);
          }
        }
        wl[qd] = pack4_lo(bl[0], bl[1], bl[2], bl[3]);
        wh[qd] = pack4_lo(bhh[0], bhh[1], bhh[2], bhh[3]);
        // v1t: tokens tb + 4 qd .. +3 (chunk tb / 8 + qd / 2, half qd & 1) and + 16 (chunk tb / 8 + 2 + qd / 2)
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          const f32x2* fg = g ? fb : fa;
          const int pos = (tb / 8 + 2 * g + (qd >> 1)) ^ (p & 7);
          uint2* r0 = reinterpret_cast<uint2*>(vst + c0 * (BC / 8) + pos) + (qd & 1);
          uint2* r1 = reinterpret_cast<uint2*>(vst + (c0 + 1) * (BC / 8) + pos) + (qd & 1);
          *r0 = make_uint2(h2of((uint32_t)fg[0], (uint32_t)fg[1]), h2of((uint32_t)fg[2], (uint32_t)fg[3]));
          *r1 = make_uint2(h2of((uint32_t)(fg[0] >> 32), (uint32_t)(fg[1] >> 32)),
                           h2of((uint32_t)(fg[2] >> 32), (uint32_t)(fg[3] >> 32)));
        }
      }
      if (bits == 4) {
        uint8_t* rv = rec + 2 * HD + u * (HD * kSub / 2) + 16 * jj;
        *reinterpret_cast<uint4*>(rv + c0 * (kSub / 2)) = make_uint4(wl[0], wl[1], wl[2], wl[3]);
        *reinterpret_cast<uint4*>(rv + (c0 + 1) * (kSub / 2)) = make_uint4(wh[0], wh[1], wh[2], wh[3]);
      } else if (BC == 128) {  // both 32-token halves of the sub-block are mine: OR them in registers
        if (gi == 0) {
#pragma unroll
          for (int qd = 0; qd < 4; ++qd) {
            wl2[qd] = wl[qd];
            wh2[qd] = wh[qd];
          }
        } else {
          uint8_t* rv = rec + 2 * HD + u * (HD * kSub / 4);
          *reinterpret_cast<uint4*>(rv + c0 * (kSub / 4)) =
              make_uint4(wl[0] | wl2[0], wl[1] | wl2[1], wl[2] | wl2[2], wl[3] | wl2[3]);
          *reinterpret_cast<uint4*>(rv + (c0 + 1) * (kSub / 4)) =
              make_uint4(wh[0] | wh2[0], wh[1] | wh2[1], wh[2] | wh2[2], wh[3] | wh2[3]);
        }
      } else {  // the two halves' bits meet in t2s (unused by V): [d][4] words of the upper half
        uint32_t* xw = reinterpret_cast<uint32_t*>(t2s);
        if (hf == 1) {
#pragma unroll
          for (int qd = 0; qd < 4; ++qd) {
            xw[c0 * 4 + qd] = wl[qd];
            xw[(c0 + 1) * 4 + qd] = wh[qd];
          }
        }
        __syncthreads();
        if (hf == 0) {
#pragma unroll
          for (int qd = 0; qd < 4; ++qd) {
            wl[qd] |= xw[c0 * 4 + qd];
            wh[qd] |= xw[(c0 + 1) * 4 + qd];
          }
          *reinterpret_cast<uint4*>(rec + 2 * HD + c0 * (kSub / 4)) = make_uint4(wl[0], wl[1], wl[2], wl[3]);
          *reinterpret_cast<uint4*>(rec + 2 * HD + (c0 + 1) * (kSub / 4)) = make_uint4(wh[0], wh[1], wh[2], wh[3]);
        }
      }
      }  // gi
    }
  } else if (kind == 0) {  // partial tail block: stage-1 outputs of its tokens only
#pragma unroll
    for (int i = 0; i < TH; ++i) {
      const f32x2 f = F(i);
      if (TH * hf + i < rows) krow[(size_t)i * (HD / 2)] = h2of((uint32_t)f, (uint32_t)(f >> 32));
    }
  } else {  // (rows past N are zero in xs: their codes are 0)
#pragma unroll
    for (int q4 = 0; q4 < TH / 8; ++q4) {
      uint32_t lo[4], hi[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const f32x2 f0 = F(8 * q4 + 2 * m), f1 = F(8 * q4 + 2 * m + 1);
        lo[m] = h2of((uint32_t)f0, (uint32_t)f1);
        hi[m] = h2of((uint32_t)(f0 >> 32), (uint32_t)(f1 >> 32));
      }
      const int pos = (TH / 8 * hf + q4) ^ (p & 7);
      vst[c0 * (BC / 8) + pos] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      vst[(c0 + 1) * (BC / 8) + pos] = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    }
  }
  __syncthreads();
  if (kind == 1) {  // V: copy the staged v1t tile out
    const uint4* tile = reinterpret_cast<const uint4*>(&xs[0][0]);
    uint4* dst = reinterpret_cast<uint4*>(v1t + (bh * Tc + j0 + j) * HD * BC);
#pragma unroll
    for (int i = tid; i < HD * BC / 8; i += HD) {
      const int r = i / (BC / 8), k8 = i % (BC / 8);
      dst[i] = tile[r * (BC / 8) + (k8 ^ ((r >> 1) & 7))];
    }
    return;
  }
  if (rows < BC) return;  // partial tail block: goes to the buffer (tail kernel)
  // K record codes from the stage-2 tile t2s [t][c] (token-major, natural channel order, LSB-first)
  const int kbits = bits_dev[h * 2];
  uint8_t* krec = block_rec + ((bh * 2) * (size_t)max_blocks + j0 + j) * REC + 2 * HD;
  if (kbits == 4) {
    for (int i = tid; i < BC * HD / 32; i += HD) {  // 32 channels (16 B of codes) per item
      const int t = i / (HD / 32), c32 = i % (HD / 32);
      const uint4 lo = *reinterpret_cast<const uint4*>(tile2 + t * HD + c32 * 32);
      const uint4 hi = *reinterpret_cast<const uint4*>(tile2 + t * HD + c32 * 32 + 16);
      *reinterpret_cast<uint4*>(krec + t * (HD / 2) + c32 * 16) =
          make_uint4(pack_nib8(make_uint2(lo.x, lo.y)), pack_nib8(make_uint2(lo.z, lo.w)),
                     pack_nib8(make_uint2(hi.x, hi.y)), pack_nib8(make_uint2(hi.z, hi.w)));
    }
  } else {
    for (int i = tid; i < BC * HD / 64; i += HD) {  // 64 channels (16 B of codes) per item
      const int t = i / (HD / 64), c64 = i % (HD / 64);
      uint32_t wv[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const uint4 u = *reinterpret_cast<const uint4*>(tile2 + t * HD + c64 * 64 + g * 16);
        wv[g] = pack_crumb8(make_uint2(u.x, u.y)) | (pack_crumb8(make_uint2(u.z, u.w)) << 16);
      }
      *reinterpret_cast<uint4*>(krec + t * (HD / 4) + c64 * 16) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    }
  }
}

template <int HD, int BC>
__global__ void __launch_bounds__(HD, (BC == 64 ? 6 : 3) * 128 / HD) quant_prefill_kernel(
    const __half* __restrict__ k, const __half* __restrict__ v, int N, int Hkv, int max_blocks, int j0, int Nk,
    const int32_t* __restrict__ bits_dev, uint8_t* __restrict__ block_rec, float* __restrict__ s_parent,
    float* __restrict__ a_univ, __half* __restrict__ k1, __half* __restrict__ v1t, float* __restrict__ k1s,
    float* __restrict__ v1s, int scale_fp16, int t0, int Nin, int8_t* __restrict__ zbuf, int32_t* __restrict__ counters) {
  // zbuf != NULL (PREFILL of a whole number of blocks): the slot's INT8 buffer is zeroed by its block-0 CTA and the
  // counters are set here -- no buffer memset and no quant_tail_kernel launch (the tail is empty).
  constexpr int NW = HD / 32;  // warps
  // One CTA per (block, kv head, batch, K or V): 6 small CTAs per SM keep more loads in
  // flight than 3 CTAs doing K and V together.  The block (FP16 [64][HD]) is staged with
  // coalesced 16-byte loads; after every thread has taken its column (the barrier of the
  // max reduction) the space is reused for K's token-major stage-1 / stage-2 code tiles.
  __shared__ __align__(16) __half xs[BC][HD];
  __shared__ float red[NW];
  // K: B_c = 64 transposes the fp16 stage-1 codes through xs (then a coalesced copy-out) and keeps the
  // stage-2 codes in t2s; B_c = 128 (48 KB static limit) writes k1 directly and keeps the stage-2 codes
  // in the second half of xs.
  __shared__ __align__(16) uint8_t t2s[BC == 64 ? BC * HD : 16];
  const int j = blockIdx.x, h = blockIdx.y, b = blockIdx.z >> 1, kind = blockIdx.z & 1, tid = threadIdx.x;
  const int rows = min(BC, N - j * BC);
  {
    constexpr int C8 = HD / 8;  // 16-byte chunks per token row
    const __half* src = kind ? v : k;
#pragma unroll
    for (int i = tid; i < BC * C8; i += HD) {
      const int t = i / C8, c8 = i % C8;
      uint4 val = make_uint4(0, 0, 0, 0);
      if (t < rows)
        val = __ldcs(reinterpret_cast<const uint4*>(src + (((size_t)b * Nin + t0 + (size_t)j * BC + t) * Hkv + h) * HD) +
                     c8);
      *reinterpret_cast<uint4*>(&xs[t][8 * c8]) = val;
    }
  }
  __syncthreads();
  quant_block<HD, BC>(xs, t2s, red, j, h, b, kind, k, v, N, Hkv, max_blocks, j0, Nk, bits_dev, block_rec, s_parent, a_univ, k1, v1t, k1s, v1s, scale_fp16, t0, Nin, zbuf, counters);
}

// Persistent: as many CTAs as fit (B_c = 64: 5 per SM, 128: 3) walk the items (kv head fastest) with the FP16
// block of the next item already on its way -- one TMA tile load ([B_c tokens][HD], the rows of one head) into
// the second buffer of a double buffer -- while the current item is quantised.
template <int HD, int BC>
constexpr size_t quant_tma_smem() { return 2 * BC * HD * 2 + (BC == 64 ? BC * HD : 0) + HD * 8 + 64; }
template <int HD, int BC>
__global__ void __launch_bounds__(HD, (BC == 64 ? 5 : 3) * 128 / HD) quant_prefill_tma_kernel(
    const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv, int n_items, int Tcn,
    const __half* __restrict__ k, const __half* __restrict__ v, int N, int Hkv, int max_blocks, int j0, int Nk,
    const int32_t* __restrict__ bits_dev, uint8_t* __restrict__ block_rec, float* __restrict__ s_parent,
    float* __restrict__ a_univ, __half* __restrict__ k1, __half* __restrict__ v1t, float* __restrict__ k1s,
    float* __restrict__ v1s, int scale_fp16, int t0, int Nin, int8_t* __restrict__ zbuf, int32_t* __restrict__ counters) {
  extern __shared__ __align__(128) uint8_t qsm[];
  __half(*xs2)[BC][HD] = reinterpret_cast<__half(*)[BC][HD]>(qsm);  // [2][B_c][HD]
  uint8_t* t2s = qsm + 2 * BC * HD * 2;                                // B_c = 64: K stage-2 codes
  uint32_t* xch = reinterpret_cast<uint32_t*>(t2s + (BC == 64 ? BC * HD : 0));  // [2][HD / 2][2] min / max
  float* red = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(xch) + HD * 8);
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + 8);
  const int tid = threadIdx.x;
  auto item = [&](int it, int& j, int& h, int& b, int& kind) {
    h = it % Hkv;
    const int r = it / Hkv;
    j = r % Tcn;
    kind = (r / Tcn) & 1;
    b = (r / Tcn) >> 1;
  };
  auto issue = [&](int it, int st) {
    int j, h, b, kind;
    item(it, j, h, b, kind);
    mbar_expect_tx(&bar[st], BC * HD * 2);  // (rows past the input are zero-filled and counted)
    tma_load_3d(&xs2[st][0][0], kind ? (const void*)&tmv : (const void*)&tmk, &bar[st], 0, h, b * Nin + t0 + j * BC);
  };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0) {
    if ((int)blockIdx.x < n_items) issue(blockIdx.x, 0);
    if ((int)(blockIdx.x + gridDim.x) < n_items) issue(blockIdx.x + gridDim.x, 1);
  }
  int i = 0;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++i) {
    const int st = i & 1;
    int j, h, b, kind;
    item(it, j, h, b, kind);
    mbar_wait(&bar[st], (i >> 1) & 1);
    const int rows = min(BC, N - j * BC);
    if (rows < BC) {  // the tile reaches past the sequence: zero those rows
      for (int e = tid; e < (BC - rows) * HD / 8; e += HD)
        reinterpret_cast<uint4*>(&xs2[st][rows][0])[e] = make_uint4(0, 0, 0, 0);
      __syncthreads();
    }
    quant_block_cp<HD, BC>(xs2[st], t2s, xch, red, j, h, b, kind, k, v, N, Hkv, max_blocks, j0, Nk, bits_dev, block_rec,
                           s_parent, a_univ, k1, v1t, k1s, v1s, scale_fp16, t0, Nin, zbuf, counters);
    __syncthreads();  // xs2[st], t2s, xch and red are free again
    if (tid == 0 && it + 2 * (int)gridDim.x < n_items) {
      fence_proxy_async();  // the generic-proxy staging writes precede the async-proxy refill
      issue(it + 2 * gridDim.x, st);
    }
  }
}


// Tail (N mod B_c tokens) -> INT8 buffer with the universal scale (R-11);
// sets the counters.  One CTA per (kv_head, batch), thread = channel x kind.
template <int HD, int BC>
__global__ void quant_tail_kernel(const __half* __restrict__ k, const __half* __restrict__ v, int N, int Hkv,
                                  const float* __restrict__ a_univ, int8_t* __restrict__ buf,
                                  int32_t* __restrict__ counters, int j0, int t0, int Nin) {
  const int h = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const int nfull = N / BC, ntail = N - nfull * BC;
  const size_t bh = (size_t)b * Hkv + h;
  if (h == 0 && tid == 0) {
    counters[b * 2 + 0] = j0 + nfull;
    counters[b * 2 + 1] = ntail;
  }
  if (tid >= 2 * HD) return;
  const int kv = tid / HD, c = tid % HD;
  const float a = a_univ[bh * 2 + kv];
  const float inv = a > 0.f ? div_119_by(a) : 0.f;
  const __half* src = kv == 0 ? k : v;
  int8_t* bslot = buf + (bh * 2 + kv) * (size_t)(BC * HD);
  for (int t = 0; t < ntail; ++t) {
    const float x = __half2float(src[(((size_t)b * Nin + t0 + (size_t)nfull * BC + t) * Hkv + h) * HD + c]);
    const int code = max(-119, min(119, rint_prod(x, inv)));
    bslot[kv == 0 ? t * HD + c : c * BC + t] = (int8_t)code;
  }
}

// APPEND one token per sequence (P:222-224 append-then-attend).
// One CTA per (kv_head, batch); thread = (kind, channel).  Flushes a full buffer.
template <int HD, int BC>
__global__ void __launch_bounds__(256) quant_append_kernel(
    const __half* __restrict__ k, const __half* __restrict__ v, int Hkv, int max_blocks,
    const int32_t* __restrict__ bits_dev, const float* __restrict__ a_univ, int8_t* __restrict__ buf,
    uint8_t* __restrict__ block_rec, float* __restrict__ s_parent, const int32_t* __restrict__ counters,
    int scale_fp16) {
  __shared__ __align__(16) int8_t tile[2][BC * HD];
  const int h = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  pdl_wait();  // (launched with PDL: the previous step's counters / buffer)
  const int n_blocks = counters[b * 2 + 0], n_buf = counters[b * 2 + 1];
  const size_t bh = (size_t)b * Hkv + h;
  const bool flush = n_buf + 1 == BC;
  if (tid < 2 * HD) {
    const int kv = tid / HD, c = tid % HD;
    const float a = a_univ[bh * 2 + kv];
    const float inv = a > 0.f ? div_119_by(a) : 0.f;
    const float x = __half2float((kv == 0 ? k : v)[bh * HD + c]);
    const int code = max(-119, min(119, rint_prod(x, inv)));
    int8_t* bslot = buf + (bh * 2 + kv) * (size_t)(BC * HD);
    bslot[kv == 0 ? n_buf * HD + c : c * BC + n_buf] = (int8_t)code;
    if (flush) {
      for (int t = 0; t < BC; ++t)
        tile[kv][t * HD + c] = t == n_buf ? (int8_t)code : bslot[kv == 0 ? t * HD + c : c * BC + t];
    }
  }
  if (!flush) return;
  if (n_blocks >= max_blocks) return;  // host checks capacity first
  __syncthreads();
  constexpr int REC = rec_bytes(HD, BC);
  uint8_t* rec[2];
#pragma unroll
  for (int kv = 0; kv < 2; ++kv) rec[kv] = block_rec + ((bh * 2 + kv) * (size_t)max_blocks + n_blocks) * REC;
  if (tid < 2 * HD) {
    const int kv = tid / HD, c = tid % HD;
    uint8_t s;
    int8_t z;
    stage2_column<BC>(tile[kv], HD, c, bits_dev[h * 2 + kv], &s, &z);
    rec[kv][c] = s;
    rec[kv][HD + c] = (uint8_t)z;
  }
  __syncthreads();
#pragma unroll
  for (int kv = 0; kv < 2; ++kv) pack_record<HD, BC>(tile[kv], kv, bits_dev[h * 2 + kv], rec[kv] + 2 * HD, tid, 256);
  if (tid < 2) s_parent[(bh * 2 + tid) * max_blocks + n_blocks] = st1_scale(div_by_119(a_univ[bh * 2 + tid]), scale_fp16);
}

__global__ void append_counters_kernel(int32_t* counters, int B, int BC) {
  pdl_wait();  // after quant_append_kernel has read the counters
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int nb = counters[b * 2], nbuf = counters[b * 2 + 1] + 1;
  if (nbuf == BC) {
    nb += 1;
    nbuf = 0;
  }
  counters[b * 2] = nb;
  counters[b * 2 + 1] = nbuf;
}

// ---------------------------------------------------------------------------
// Stage-1 reconstruction of cache blocks (chunked prefill, R-28): block j of
// (b, kv head) -> k1 rows [B_c j, B_c j + B_c) and v1t block j of the prefill
// operand layout, values code s_int + z_int (Alg. 2; exact in int8,
// R-6), scales = the blocks' parent scales.  One CTA per (block, kv head,
// batch), thread = (K/V, channel).
template <int HD, int BC>
__global__ void __launch_bounds__(2 * HD) dequant_cache_kernel(
    int Hkv, int max_blocks, int blk_begin, int blk_end, int Nk, const int32_t* __restrict__ bits_dev,
    const uint8_t* __restrict__ block_rec, const float* __restrict__ s_parent, const int32_t* __restrict__ counters,
    __half* __restrict__ k1, __half* __restrict__ v1t, float* __restrict__ k1s, float* __restrict__ v1s) {
  const int j = blk_begin + blockIdx.x, h = blockIdx.y, b = blockIdx.z, tid = threadIdx.x;
  const int nb = counters[b * 2];
  if (j >= nb || (blk_end >= 0 && j >= blk_end)) return;
  const int kind = tid / HD, c = tid % HD, Tk = (Nk + BC - 1) / BC;
  const size_t bh = (size_t)b * Hkv + h;
  const int bits = bits_dev[h * 2 + kind];
  constexpr int REC = rec_bytes(HD, BC);
  const uint8_t* rec = block_rec + ((bh * 2 + kind) * (size_t)max_blocks + j) * REC;
  const int sc = rec[c], zc = (int)(int8_t)rec[HD + c];
  const uint8_t* codes = rec + 2 * HD;
  const uint32_t mask = (1u << bits) - 1u;
  if (tid % HD == 0) (kind ? v1s : k1s)[bh * Tk + j] = s_parent[(bh * 2 + kind) * max_blocks + j];
  if (kind == 0) {
    // K: token-major, channel c in byte c bits / 8 at bit (c bits) % 8 (layout.cuh)
    const int TB = HD * bits / 8, byte = c * bits / 8, sh = (c * bits) % 8;
#pragma unroll 4
    for (int t = 0; t < BC; ++t)
      k1[(bh * Nk + (size_t)j * BC + t) * HD + c] = __int2half_rn((int)((codes[t * TB + byte] >> sh) & mask) * sc + zc);
  } else {
    // V: channel-major words per 64-token sub-block in the IMMA token order (layout.cuh v_token_of)
    const int CB = kSub * bits / 8;
    __align__(16) __half row[BC];  // read back as uint4 below
    for (int u = 0; u < BC / kSub; ++u)
      for (int wi = 0; wi < CB / 4; ++wi)
        for (int i = 0; i < 32 / bits; ++i) {
          int e, sh;
          const int t = kSub * u + v_token_of(bits, wi, i, &e, &sh);
          row[t] = __int2half_rn((int)((codes[u * HD * CB + c * CB + 4 * wi + e] >> sh) & mask) * sc + zc);
        }
    uint4* dst = reinterpret_cast<uint4*>(v1t + ((bh * Tk + j) * HD + c) * BC);
#pragma unroll
    for (int t8 = 0; t8 < BC / 8; ++t8) dst[t8] = reinterpret_cast<const uint4*>(row)[t8];
  }
}

// ---------------------------------------------------------------------------
// R-31: a prefill chunk into a cache that ends inside a block (cache block j0 holds nbuf buffered
// tokens): its first r tokens complete that block exactly as APPEND does -- universal-scale codes,
// clamped to +-119, into buffer rows nbuf .. nbuf + r - 1 -- and, as the chunk's stage-1 operands,
// into k1 rows B_c j0 + nbuf + t and v1t block j0 columns nbuf + t; a full block is flushed
// (stage 2, parent s_univ).  One CTA per (kv head, batch); thread = (K/V, channel).
template <int HD, int BC>
__global__ void __launch_bounds__(256) quant_boundary_kernel(
    const __half* __restrict__ k, const __half* __restrict__ v, int N, int r, int Hkv, int max_blocks, int j0, int nbuf,
    int Nk, const int32_t* __restrict__ bits_dev, const float* __restrict__ a_univ, int8_t* __restrict__ buf,
    uint8_t* __restrict__ block_rec, float* __restrict__ s_parent, __half* __restrict__ k1, __half* __restrict__ v1t,
    int scale_fp16) {
  __shared__ __align__(16) int8_t tile[2][BC * HD];
  const int h = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const size_t bh = (size_t)b * Hkv + h;
  const int Tk = (Nk + BC - 1) / BC;
  const bool flush = nbuf + r == BC;
  if (tid < 2 * HD) {
    const int kv = tid / HD, c = tid % HD;
    const float a = a_univ[bh * 2 + kv];
    const float inv = a > 0.f ? div_119_by(a) : 0.f;
    const __half* src = kv == 0 ? k : v;
    int8_t* bslot = buf + (bh * 2 + kv) * (size_t)(BC * HD);
    for (int t = 0; t < r; ++t) {
      const float x = __half2float(src[(((size_t)b * N + t) * Hkv + h) * HD + c]);
      const int code = max(-119, min(119, rint_prod(x, inv)));
      const int row = nbuf + t;
      bslot[kv == 0 ? row * HD + c : c * BC + row] = (int8_t)code;
      if (kv == 0) k1[(bh * Nk + (size_t)j0 * BC + row) * HD + c] = __int2half_rn(code);
      else v1t[((bh * Tk + j0) * HD + c) * BC + row] = __int2half_rn(code);
    }
    if (flush)
      for (int t = 0; t < BC; ++t) tile[kv][t * HD + c] = bslot[kv == 0 ? t * HD + c : c * BC + t];
  }
  if (!flush || j0 >= max_blocks) return;  // (the host checks capacity first)
  __syncthreads();
  constexpr int REC = rec_bytes(HD, BC);
  uint8_t* rec[2];
#pragma unroll
  for (int kv = 0; kv < 2; ++kv) rec[kv] = block_rec + ((bh * 2 + kv) * (size_t)max_blocks + j0) * REC;
  if (tid < 2 * HD) {
    const int kv = tid / HD, c = tid % HD;
    uint8_t s;
    int8_t z;
    stage2_column<BC>(tile[kv], HD, c, bits_dev[h * 2 + kv], &s, &z);
    rec[kv][c] = s;
    rec[kv][HD + c] = (uint8_t)z;
  }
  __syncthreads();
#pragma unroll
  for (int kv = 0; kv < 2; ++kv) pack_record<HD, BC>(tile[kv], kv, bits_dev[h * 2 + kv], rec[kv] + 2 * HD, tid, 256);
  if (tid < 2) s_parent[(bh * 2 + tid) * max_blocks + j0] = st1_scale(div_by_119(a_univ[bh * 2 + tid]), scale_fp16);
}

__global__ void boundary_counters_kernel(int32_t* counters, int B, int BC, int r) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int nb = counters[b * 2], nbuf = counters[b * 2 + 1] + r;
  if (nbuf == BC) {
    nb += 1;
    nbuf = 0;
  }
  counters[b * 2] = nb;
  counters[b * 2 + 1] = nbuf;
}

// The buffered tokens as the prefill operands of the boundary block (R-31): k1 rows B_c nb + t and
// v1t block nb columns t < n_buf (the rest of the block's columns 0), scales s_univ.  One CTA per
// (kv head, batch); thread = (K/V, channel).
template <int HD, int BC>
__global__ void __launch_bounds__(2 * HD) dequant_buffer_kernel(int Hkv, int Nk, const int8_t* __restrict__ buf,
                                                               const float* __restrict__ a_univ,
                                                               const int32_t* __restrict__ counters,
                                                               __half* __restrict__ k1, __half* __restrict__ v1t,
                                                               float* __restrict__ k1s, float* __restrict__ v1s,
                                                               int scale_fp16) {
  const int h = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const int nb = counters[b * 2], nbuf = counters[b * 2 + 1];
  if (nbuf == 0) return;
  const int kind = tid / HD, c = tid % HD, Tk = (Nk + BC - 1) / BC;
  const size_t bh = (size_t)b * Hkv + h;
  const int8_t* bslot = buf + (bh * 2 + kind) * (size_t)(BC * HD);
  if (c == 0) (kind ? v1s : k1s)[bh * Tk + nb] = st1_scale(div_by_119(a_univ[bh * 2 + kind]), scale_fp16);
  if (kind == 0) {
    for (int t = 0; t < nbuf; ++t) k1[(bh * Nk + (size_t)nb * BC + t) * HD + c] = __int2half_rn((int)bslot[t * HD + c]);
  } else {
    for (int t = 0; t < BC; ++t)
      v1t[((bh * Tk + nb) * HD + c) * BC + t] = __int2half_rn(t < nbuf ? (int)bslot[c * BC + t] : 0);
  }
}

}  // namespace ta

// ---------------------------------------------------------------------------
// Host launchers (called from api.cu after validation).
namespace ta_host {
using namespace ta;

template <int HD, int BC>
static void quant_boundary_hd(const turbo_kv_cache_t* c, const __half* k, const __half* v, int N, int r, int j0,
                              int nbuf, int Nk, __half* k1, __half* v1t, cudaStream_t st, int scale_fp16) {
  quant_boundary_kernel<HD, BC><<<dim3(c->n_kv_heads, c->batch), 256, 0, st>>>(
      k, v, N, r, c->n_kv_heads, c->max_blocks, j0, nbuf, Nk, c->bits_dev, c->a_univ, c->buf, c->block_rec,
      c->s_parent, k1, v1t, scale_fp16);
  boundary_counters_kernel<<<(c->batch + 127) / 128, 128, 0, st>>>(c->counters, c->batch, BC, r);
}

typedef CUresult (*EncodeTiledQFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
// FP16 K or V input [tokens][Hkv][HD] as a 3-D map (HD, Hkv, tokens); box = the B_c rows of one head.
static bool make_rows_map(CUtensorMap* m, const __half* base, int HD, int H, uint64_t tokens, int BC) {
  static const EncodeTiledQFn enc = [] {  // (thread-safe one-time init)
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess) fn = nullptr;
    return reinterpret_cast<EncodeTiledQFn>(fn);
  }();
  if (!enc) return false;
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
  cuuint64_t dims[3] = {(cuuint64_t)HD, (cuuint64_t)H, tokens};
  cuuint64_t strides[2] = {(cuuint64_t)HD * 2, (cuuint64_t)H * HD * 2};
  cuuint32_t box[3] = {(cuuint32_t)HD, 1, (cuuint32_t)BC};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<__half*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int HD, int BC>
static void quant_prefill_hd(const turbo_kv_cache_t* c, const __half* k, const __half* v, int N, __half* k1,
                             __half* v1t, float* k1s, float* v1s, cudaStream_t st, int j0, int Nk, int scale_fp16,
                             int t0, int Nin) {
  const int B = c->batch, H = c->n_kv_heads, Tc = (N + BC - 1) / BC;
  dim3 grid(Tc, H, 2 * B);  // z = 2 b + (K, V)
  // PREFILL of whole blocks (no tail): the kernel zeroes the buffer and sets the counters itself
  const bool whole = Nk == N && j0 == 0 && t0 == 0 && N % BC == 0;
  int8_t* zbuf = whole ? c->buf : nullptr;
  CUtensorMap tmk, tmv;
  if (!getenv("TURBO_QUANT_NOTMA") && make_rows_map(&tmk, k, HD, H, (uint64_t)B * Nin, BC) &&
      make_rows_map(&tmv, v, HD, H, (uint64_t)B * Nin, BC)) {
    constexpr size_t smem = quant_tma_smem<HD, BC>();
    // resident CTAs of this instantiation (thread-safe one-time init; one device per process)
    static const int resident = [] {
      int dev = 0, sms = 0, per_sm = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaFuncSetAttribute(quant_prefill_tma_kernel<HD, BC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, quant_prefill_tma_kernel<HD, BC>, HD, smem);
      return sms * std::max(1, per_sm);
    }();
    const int n_items = Tc * H * 2 * B;
    const int ctas = std::max(1, std::min(n_items, resident));
    quant_prefill_tma_kernel<HD, BC><<<ctas, HD, smem, st>>>(tmk, tmv, n_items, Tc, k, v, N, H, c->max_blocks, j0,
                                                             Nk, c->bits_dev, c->block_rec, c->s_parent, c->a_univ,
                                                             k1, v1t, k1s, v1s, scale_fp16, t0, Nin, zbuf,
                                                             c->counters);
  } else {
    quant_prefill_kernel<HD, BC><<<grid, HD, 0, st>>>(k, v, N, H, c->max_blocks, j0, Nk, c->bits_dev, c->block_rec,
                                                     c->s_parent, c->a_univ, k1, v1t, k1s, v1s, scale_fp16, t0, Nin,
                                                     zbuf, c->counters);
  }
  if (!whole)
    quant_tail_kernel<HD, BC><<<dim3(H, B), 256, 0, st>>>(k, v, N, H, c->a_univ, c->buf, c->counters, j0, t0, Nin);
}

cudaError_t launch_quant_prefill(const turbo_kv_cache_t* c, const __half* k, const __half* v, int N, __half* k1,
                                 __half* v1t, float* k1s, float* v1s, cudaStream_t st, int j0, int Nk,
                                 int scale_fp16) {
  // j0 = 0, Nk = N: PREFILL (resets the universal scales and the buffer); j0 > 0: a
  // further prefill chunk appended at cache block j0 (R-28), stage-1 outputs over Nk tokens.
  // A chunk into a cache that ends inside a block (n_buf = Nk - N - B_c j0 > 0, R-31) first
  // completes that block as appends do (quant_boundary_kernel), the rest is block-aligned.
  const int B = c->batch, H = c->n_kv_heads, HD = c->head_dim, BC = c->block_kv;
  cudaError_t e = cudaSuccess;
  if (Nk == N) {  // PREFILL (no cached tokens before)
    e = cudaMemsetAsync(c->a_univ, 0, sizeof(float) * B * H * 2, st);
    if (e != cudaSuccess) return e;
    if (N % BC != 0) {  // (a whole number of blocks: quant_prefill_kernel zeroes the buffer)
      e = cudaMemsetAsync(c->buf, 0, (size_t)B * H * 2 * BC * HD, st);
      if (e != cudaSuccess) return e;
    }
  }
  int t0 = 0;
  const int nbuf = (Nk - N) - j0 * BC;  // buffered tokens before the chunk (R-31)
  if (nbuf > 0) {
    const int r = std::min(N, BC - nbuf);
    if (HD == 128) {
      if (BC == 64) quant_boundary_hd<128, 64>(c, k, v, N, r, j0, nbuf, Nk, k1, v1t, st, scale_fp16);
      else quant_boundary_hd<128, 128>(c, k, v, N, r, j0, nbuf, Nk, k1, v1t, st, scale_fp16);
    } else {
      if (BC == 64) quant_boundary_hd<64, 64>(c, k, v, N, r, j0, nbuf, Nk, k1, v1t, st, scale_fp16);
      else quant_boundary_hd<64, 128>(c, k, v, N, r, j0, nbuf, Nk, k1, v1t, st, scale_fp16);
    }
    if (r == N) return cudaGetLastError();
    t0 = r;  // the rest starts the next block
    j0 += 1;
  }
  const int n = N - t0;
  if (HD == 128) {
    if (BC == 64) quant_prefill_hd<128, 64>(c, k, v, n, k1, v1t, k1s, v1s, st, j0, Nk, scale_fp16, t0, N);
    else quant_prefill_hd<128, 128>(c, k, v, n, k1, v1t, k1s, v1s, st, j0, Nk, scale_fp16, t0, N);
  } else {
    if (BC == 64) quant_prefill_hd<64, 64>(c, k, v, n, k1, v1t, k1s, v1s, st, j0, Nk, scale_fp16, t0, N);
    else quant_prefill_hd<64, 128>(c, k, v, n, k1, v1t, k1s, v1s, st, j0, Nk, scale_fp16, t0, N);
  }
  return cudaGetLastError();
}

template <int HD, int BC>
static void dequant_cache_hd(const turbo_kv_cache_t* c, dim3 grid, int blk_begin, int blk_end, int Nk, __half* k1,
                             __half* v1t, float* k1s, float* v1s, cudaStream_t st) {
  dequant_cache_kernel<HD, BC><<<grid, 2 * HD, 0, st>>>(c->n_kv_heads, c->max_blocks, blk_begin, blk_end, Nk,
                                                        c->bits_dev, c->block_rec, c->s_parent, c->counters, k1, v1t,
                                                        k1s, v1s);
}

cudaError_t launch_dequant_cache(const turbo_kv_cache_t* c, int blk_begin, int blk_end, int Nk, __half* k1,
                                 __half* v1t, float* k1s, float* v1s, cudaStream_t st, int scale_fp16) {
  const int B = c->batch, H = c->n_kv_heads, HD = c->head_dim, BC = c->block_kv;
  const int last = blk_end >= 0 ? std::min(blk_end, c->max_blocks) : c->max_blocks;
  dim3 grid(std::max(0, last - blk_begin), H, B);
  if (last > blk_begin) {
    if (HD == 128) {
      if (BC == 64) dequant_cache_hd<128, 64>(c, grid, blk_begin, blk_end, Nk, k1, v1t, k1s, v1s, st);
      else dequant_cache_hd<128, 128>(c, grid, blk_begin, blk_end, Nk, k1, v1t, k1s, v1s, st);
    } else {
      if (BC == 64) dequant_cache_hd<64, 64>(c, grid, blk_begin, blk_end, Nk, k1, v1t, k1s, v1s, st);
      else dequant_cache_hd<64, 128>(c, grid, blk_begin, blk_end, Nk, k1, v1t, k1s, v1s, st);
    }
  }
  if (blk_end < 0 && c->n_tokens % BC != 0) {  // the buffered tail as the boundary block (R-31)
    const dim3 g2(H, B);
    if (HD == 128) {
      if (BC == 64)
        dequant_buffer_kernel<128, 64><<<g2, 256, 0, st>>>(H, Nk, c->buf, c->a_univ, c->counters, k1, v1t, k1s, v1s, scale_fp16);
      else
        dequant_buffer_kernel<128, 128><<<g2, 256, 0, st>>>(H, Nk, c->buf, c->a_univ, c->counters, k1, v1t, k1s, v1s, scale_fp16);
    } else {
      if (BC == 64)
        dequant_buffer_kernel<64, 64><<<g2, 128, 0, st>>>(H, Nk, c->buf, c->a_univ, c->counters, k1, v1t, k1s, v1s, scale_fp16);
      else
        dequant_buffer_kernel<64, 128><<<g2, 128, 0, st>>>(H, Nk, c->buf, c->a_univ, c->counters, k1, v1t, k1s, v1s, scale_fp16);
    }
  }
  return cudaGetLastError();
}

template <int HD, int BC>
static void quant_append_hd(const turbo_kv_cache_t* c, const __half* k, const __half* v, cudaStream_t st,
                            int scale_fp16) {
  launch_pdl(quant_append_kernel<HD, BC>, dim3(c->n_kv_heads, c->batch), dim3(256), 0, st, k, v, c->n_kv_heads,
             c->max_blocks, (const int32_t*)c->bits_dev, (const float*)c->a_univ, c->buf, c->block_rec, c->s_parent,
             (const int32_t*)c->counters, scale_fp16);
}

cudaError_t launch_quant_append(const turbo_kv_cache_t* c, const __half* k, const __half* v, cudaStream_t st,
                                int scale_fp16) {
  const int B = c->batch, HD = c->head_dim, BC = c->block_kv;
  if (HD == 128) {
    if (BC == 64) quant_append_hd<128, 64>(c, k, v, st, scale_fp16);
    else quant_append_hd<128, 128>(c, k, v, st, scale_fp16);
  } else {
    if (BC == 64) quant_append_hd<64, 64>(c, k, v, st, scale_fp16);
    else quant_append_hd<64, 128>(c, k, v, st, scale_fp16);
  }
  launch_pdl(append_counters_kernel, dim3((B + 127) / 128), dim3(128), 0, st, c->counters, B, BC);
  return cudaGetLastError();
}
}  // namespace ta_host
