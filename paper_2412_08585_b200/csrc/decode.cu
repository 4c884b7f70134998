// decode.cu -- Algorithm 2 (TurboAttention decode) on sm_100a,
// plus the split-KV log-sum-exp combine (R-23).
//
// One WARP (= one CTA) = one (batch, kv head, split) task, or one chunk of the
// balanced schedule; it owns the G = Hq/Hkv query rows of that KV head (GQA,
// R-22) and walks its contiguous block range in Alg. 2 order.  Block records (s_int | z_int | packed codes) stream through a
// per-warp 2-stage smem ring with cp.async.bulk (TMA 1-D) + mbarrier; codes are
// unpacked in registers straight into mma.sync m16n8k32 IMMA fragments.
//
// Integer dequantisation (Alg. 2) is folded exactly (Eq. 5, P:275-283,
// linear because reconstructions never clamp, R-6):
//   S[t]    = sum_c q1_c (code_tc s_c + z_c)
//           = 256 * sum_c hi(q1_c s_c) code_tc + sum_c lo(q1_c s_c) code_tc + sum_c q1_c z_c
//   PV[c]   = sum_t P_t (code_tc s_c + z_c) = s_c * sum_t P_t code_tc + z_c * sum_t P_t
// with q1_c s_c = 256 hi + lo, lo = the signed low byte, hi in [-38, 37] (both s8), so the
// tensor cores see only raw 4-bit / 2-bit codes.
#include <algorithm>
#include <climits>
#include <cstring>

#include "common.cuh"
#include "layout.cuh"

namespace ta {

// One warp per CTA: a finished task frees its SM slot at once (the block
// scheduler refills it), instead of holding it until the CTA's slowest warp
// ends -- +3-6 % KV GB/s on configs[2] / configs[4] and far less sensitivity
// to the split count (tools/sweep_decode.py).
constexpr int kWarpsPerCta = 1;
constexpr int kMinUnits = 8;  // balanced schedule: least units (blocks) per warp chunk

// Per-warp shared memory.  ROWS = query rows held (G <= 4 on the packed path,
// else 8), so that twelve packed-path warps fit in one SM's 228 KB.
template <int HD, int ROWS, int BC>
struct DecodeWarpSmem {
  uint8_t rec[2][2][rec_bytes(HD, BC)];  // [stage][K,V][record]
  int8_t q1[ROWS][HD];
  uint8_t p[ROWS][BC];
  uint64_t bar[2];
};
template <int HD, bool PACK, int BC>
using DecodeSmem = DecodeWarpSmem<HD, PACK ? 4 : 8, BC>;

struct DecodeArgs {
  const __half* q;
  const uint8_t* block_rec;
  const float* s_parent;
  const int8_t* buf;
  const float* a_univ;
  const int32_t* counters;
  const int32_t* bits;
  float* o_parts;   // [S][B][Hq][d]  (or the final f32 output when S == 1)
  float* lse_parts; // [S][B][Hq]
  __half* o16;      // final fp16 output when S == 1 (or NULL)
  __half* fin_o16;  // balanced schedule: final fp16 output (or NULL)
  float* fin_o32;   // balanced schedule: final f32 output (or NULL)
  float* fin_lse;   // balanced schedule: final L
  // Hkv and G are VIRTUAL when the group has more than 8 query rows: each KV head's G_real rows are cut into RG
  // row groups of G = G_real / RG rows (virtual KV head vk = kvh RG + rg, query head vk G + row as before), so a
  // task holds at most 8 rows; the cache slot is (b, vk / RG).
  int B, Hq, Hkv, G, RG, max_blocks, blk_begin, blk_end, with_buffer, n_splits, alpha_mode, scale_fp16, sas_fp16;
  float scale;
  SasConst sas;
  turbo_debug_tap_t tap;
};

TA_DEV uint32_t word_of(const uint4& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }
TA_DEV uint32_t byte_of(const uint4& v, int i) {  // one PRMT (i is a compile-time constant)
  const uint32_t w = i < 4 ? v.x : i < 8 ? v.y : i < 12 ? v.z : v.w;
  return __byte_perm(w, 0u, 0x4440u | (uint32_t)(i & 3));
}

// Shared-memory accessors on 32-bit shared addresses.
TA_DEV uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
TA_DEV uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
TA_DEV uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
TA_DEV int lds_s8(uint32_t a) {
  int v;
  asm volatile("ld.shared.s8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
TA_DEV void sts_u8(uint32_t a, uint32_t v) { asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
// N consecutive 32-bit words from a 4N-byte aligned shared address (one LDS.32/64/128).
template <int N>
TA_DEV void lds_words(uint32_t a, uint32_t (&w)[N]) {
  if (N == 4) {
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(w[0]), "=r"(w[N > 1 ? 1 : 0]), "=r"(w[N > 2 ? 2 : 0]),
                 "=r"(w[N > 3 ? 3 : 0]) : "r"(a));
  } else if (N == 2) {
    asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(w[0]), "=r"(w[N > 1 ? 1 : 0]) : "r"(a));
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) asm volatile("ld.shared.b32 %0, [%1];" : "=r"(w[i]) : "r"(a + 4 * i));
  }
}

// Reductions over the lanes that hold the same two query rows: general path
// (rows 2q, 2q+1): lanes with equal q; packed path (rows 2(q&1), +1): equal q&1.
template <bool PACK>
TA_DEV float grp_maxf(float v) {
  if (PACK) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <bool PACK>
TA_DEV float grp_sumf(float v) {
  if (PACK) v += __shfl_xor_sync(0xffffffffu, v, 2);
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <bool PACK>
TA_DEV int grp_maxi(int v) {
  if (PACK) v = max(v, __shfl_xor_sync(0xffffffffu, v, 2));
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <bool PACK>
TA_DEV int grp_sumi(int v) {
  if (PACK) v += __shfl_xor_sync(0xffffffffu, v, 2);
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// K codes are consumed without shifting them down: 4-bit codes as the masked
// nibbles (w & 0x0F0F0F0F) and 16 x (w & 0xF0F0F0F0), 2-bit codes as
// 4^s x ((w >> 2s) & 3) -- each "unit" (one scale) gets its own IMMA
// accumulator and the exact sum is  sum_u acc_u >> (log2 scale_u).
// Unit u, B register r (0: k-slots 4q+m, 1: k-slots 16+4q+m), slot m -> the
// channel inside the lane quad's K region (layout.cuh: byte b of a token holds
// channels b*8/bits ...), or -1 for a zero slot (d = 64, 2-bit).
template <int HD, int BITS>
struct KUnits {
  static constexpr int QB = HD * BITS / 32;             // bytes of a token's lane-quad region
  static constexpr int NW = QB / 4;                     // 32-bit words per region
  static constexpr int N = BITS == 4 ? NW : 4;          // units: 4-bit (word pair, lo/hi); 2-bit: s = 0..3
  TA_DEV static constexpr int chan(int u, int r, int m) {
    if (BITS == 4) {
      const int pair = u >> 1, half = u & 1;
      return 8 * (2 * pair + r) + 2 * m + half;
    }
    return (r == 1 && NW < 2) ? -1 : 16 * r + 4 * m + u;
  }
  TA_DEV static constexpr int shift(int u) { return BITS == 4 ? 4 * (u & 1) : 2 * u; }
  TA_DEV static uint32_t mask(int u) { return BITS == 4 ? ((u & 1) ? 0xF0F0F0F0u : 0x0F0F0F0Fu) : (0x03030303u << (2 * u)); }
  // word index (inside the region) feeding A register r of unit u
  TA_DEV static constexpr int word(int u, int r) { return BITS == 4 ? 2 * (u >> 1) + r : r; }
};

// Thread <-> data maps.  Lane = 4 g + q.
//   General path (G <= 8): rows 2q+e; score values t = 2 mt + h at token
//   16 mt + g + 8 h (NT = 8); O values c = 2 mt + h at channel 16 mt + g + 8 h.
//   Packed path (G <= 4): the 4 spare MMA columns carry the lo half of the
//   Eq. 5 fold, rows 2(q&1)+e; t = mt at token 16 mt + g + 8 (q>>1) (NT = 4);
//   O values c = mt at channel 16 mt + g + 8 (q>>1).
template <int HD, bool PACK>
struct Map {
  static constexpr int NT = PACK ? 4 : 8;
  static constexpr int NC = PACK ? HD / 16 : HD / 8;
  TA_DEV static int row(int q, int e) { return PACK ? 2 * (q & 1) + e : 2 * q + e; }
  TA_DEV static int tok(int t, int g, int q) { return PACK ? 16 * t + g + 8 * (q >> 1) : 16 * (t >> 1) + g + 8 * (t & 1); }
  TA_DEV static int chan(int c, int g, int q) { return PACK ? 16 * c + g + 8 * (q >> 1) : 16 * (c >> 1) + g + 8 * (c & 1); }
};

// QK^T on a stage-2 block (Alg. 2, folded): S_int per thread value.
template <int HD, int BK, bool PACK, int BC>
TA_DEV void qk_block(uint32_t rec, const int (&qv)[HD / 4], const uint4 (&q1r)[HD / 64],
                     int (&sv)[Map<HD, PACK>::NT * BC / 64][2], int g, int q) {
  using U = KUnits<HD, BK>;
  constexpr int R = HD / 4;
  uint4 s4[HD / 64];
#pragma unroll
  for (int i = 0; i < HD / 64; ++i) s4[i] = lds128(rec + q * R + 16 * i);
  // B fragments from q1_c * s_c = 256 hi + lo (lo = signed low byte, hi = (q1_c s_c + 128) >> 8,
  // both s8).  With t = q1_c s_c + 128 from one IDP.4A (s word . q1_c placed in byte c mod 4,
  // accumulator 128): hi = byte 1 of t, lo = byte 0 of t ^ 0x80 -- byte selects only.  Packed
  // path: column g < 4 holds hi of row g, column g >= 4 holds lo of row g - 4 (one IMMA);
  // general path: separate hi and lo IMMAs.
  const uint32_t psel = (PACK && g >= 4) ? 0x40u : 0x51u;  // PRMT pair select: byte 0 / byte 1
  const uint32_t pxor = (PACK && g >= 4) ? 0x80808080u : 0u;
  uint32_t bhi[U::N][2], blo[U::N][2];
#pragma unroll
  for (int u = 0; u < U::N; ++u)
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      uint32_t t[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int loc = U::chan(u, r, m);  // zero slot: t = 128 -> hi = lo = 0
        t[m] = loc < 0 ? 128u : (uint32_t)__dp4a((int)word_of(s4[loc >> 4], (loc & 15) >> 2), qv[loc], 128);
      }
      bhi[u][r] = __byte_perm(__byte_perm(t[0], t[1], psel), __byte_perm(t[2], t[3], psel), 0x5410) ^ pxor;
      if (!PACK)
        blo[u][r] = __byte_perm(__byte_perm(t[0], t[1], 0x40), __byte_perm(t[2], t[3], 0x40), 0x5410) ^ 0x80808080u;
    }
  // z term sum_c q1_c z_c of the lane-quad's row (dp4a, quad reduction).
  int zq = 0;
#pragma unroll
  for (int i = 0; i < HD / 64; ++i) {
    const uint4 zv = lds128(rec + HD + q * R + 16 * i);
    zq = __dp4a((int)zv.x, (int)q1r[i].x, zq);
    zq = __dp4a((int)zv.y, (int)q1r[i].y, zq);
    zq = __dp4a((int)zv.z, (int)q1r[i].z, zq);
    zq = __dp4a((int)zv.w, (int)q1r[i].w, zq);
  }
  zq += __shfl_xor_sync(0xffffffffu, zq, 1);
  zq += __shfl_xor_sync(0xffffffffu, zq, 2);
  const int rq = PACK ? (q & 1) : q;
  const int z0 = __shfl_sync(0xffffffffu, zq, 8 * rq), z1 = __shfl_sync(0xffffffffu, zq, 8 * rq + 4);
  // A fragments: masked (unshifted) codes of tokens 16 mt + g (+8).
  constexpr int TB = HD * BK / 8;
  const uint32_t codes = rec + 2 * HD;
#pragma unroll
  for (int mt = 0; mt < BC / 16; ++mt) {
    uint32_t w0[U::NW], w1[U::NW];
    const uint32_t t0 = codes + (16 * mt + g) * TB + q * U::QB, t1 = t0 + 8 * TB;
    lds_words<U::NW>(t0, w0);  // one vector load per token region
    lds_words<U::NW>(t1, w1);
    int ch[4] = {0, 0, 0, 0}, cl[4] = {0, 0, 0, 0};
    if (!PACK) {
      // (the z term starts the lo accumulators: S = 256 hi + lo + sum q1 z)
      cl[0] = cl[2] = z0;
      cl[1] = cl[3] = z1;
      // General path (G > 4, issue-bound): the IMMAs accumulate in place.  4-bit: the low-nibble units
      // straight into ch / cl, the high-nibble units (codes x 16) into a second pair, shifted back once;
      // 2-bit: the code words are shifted down first, so every unit has scale 1.
      int ch16[4] = {0, 0, 0, 0}, cl16[4] = {0, 0, 0, 0};
#pragma unroll
      for (int u = 0; u < U::N; ++u) {
        uint32_t af[4];
        const int sh = BK == 4 ? 0 : U::shift(u);
        const uint32_t mk = BK == 4 ? U::mask(u) : 0x03030303u;
        af[0] = (w0[U::word(u, 0)] >> sh) & mk;
        af[1] = (w1[U::word(u, 0)] >> sh) & mk;
        af[2] = U::chan(u, 1, 0) < 0 ? 0u : (w0[U::word(u, 1) < U::NW ? U::word(u, 1) : 0] >> sh) & mk;
        af[3] = U::chan(u, 1, 0) < 0 ? 0u : (w1[U::word(u, 1) < U::NW ? U::word(u, 1) : 0] >> sh) & mk;
        const uint32_t bh[2] = {bhi[u][0], bhi[u][1]}, bl[2] = {blo[u][0], blo[u][1]};
        if (BK == 4 && U::shift(u) != 0) {
          imma_u8s8(ch16, af, bh);
          imma_u8s8(cl16, af, bl);
        } else {
          imma_u8s8(ch, af, bh);
          imma_u8s8(cl, af, bl);
        }
      }
      if (BK == 4) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          ch[i] += ch16[i] >> 4;  // exact: a multiple of 16
          cl[i] += cl16[i] >> 4;
        }
      }
    } else {
#pragma unroll
    for (int u = 0; u < U::N; ++u) {
      int cu[4] = {0, 0, 0, 0};
      uint32_t af[4];
      const uint32_t mk = U::mask(u);
      af[0] = w0[U::word(u, 0)] & mk;
      af[1] = w1[U::word(u, 0)] & mk;
      af[2] = U::chan(u, 1, 0) < 0 ? 0u : w0[U::word(u, 1) < U::NW ? U::word(u, 1) : 0] & mk;
      af[3] = U::chan(u, 1, 0) < 0 ? 0u : w1[U::word(u, 1) < U::NW ? U::word(u, 1) : 0] & mk;
      const uint32_t bh[2] = {bhi[u][0], bhi[u][1]};
      imma_u8s8(cu, af, bh);
#pragma unroll
      for (int i = 0; i < 4; ++i) ch[i] += cu[i] >> U::shift(u);  // exact: acc_u is a multiple of its scale
    }
    }
    if (PACK) {
      // exchange hi / lo halves between lane quads q and q ^ 2
      const bool ql = q >= 2;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int own = ql ? ch[2 + e] : ch[e];
        const int snd = ql ? ch[e] : ch[2 + e];
        const int rcv = __shfl_xor_sync(0xffffffffu, snd, 2);
        const int hi = ql ? rcv : own, lo = ql ? own : rcv;
        sv[mt][e] = 256 * hi + lo + (e ? z1 : z0);
      }
    } else {
      sv[2 * mt][0] = 256 * ch[0] + cl[0];
      sv[2 * mt][1] = 256 * ch[1] + cl[1];
      sv[2 * mt + 1][0] = 256 * ch[2] + cl[2];
      sv[2 * mt + 1][1] = 256 * ch[3] + cl[3];
    }
  }
}

// QK^T on the INT8 buffer block (token-major K, natural channels; s8 x s8).
template <int HD, bool PACK, int BC>
TA_DEV void qk_buffer(const int8_t* kb, uint32_t q1s, int (&sv)[Map<HD, PACK>::NT * BC / 64][2], int g, int q) {
  const int rn = PACK ? (g & 3) : g;
#pragma unroll
  for (int mt = 0; mt < BC / 16; ++mt) {
    int c[4] = {0, 0, 0, 0};
    const int t0 = 16 * mt + g, t1 = t0 + 8;
#pragma unroll
    for (int j = 0; j < HD / 32; ++j) {
      uint32_t af[4];
      af[0] = *reinterpret_cast<const uint32_t*>(kb + t0 * HD + 32 * j + 4 * q);
      af[1] = *reinterpret_cast<const uint32_t*>(kb + t1 * HD + 32 * j + 4 * q);
      af[2] = *reinterpret_cast<const uint32_t*>(kb + t0 * HD + 32 * j + 16 + 4 * q);
      af[3] = *reinterpret_cast<const uint32_t*>(kb + t1 * HD + 32 * j + 16 + 4 * q);
      const uint32_t bq[2] = {lds32(q1s + rn * HD + 32 * j + 4 * q), lds32(q1s + rn * HD + 32 * j + 16 + 4 * q)};
      imma_s8s8(c, af, bq);
    }
    if (PACK) {
      const bool ql = q >= 2;
      sv[mt][0] = ql ? c[2] : c[0];
      sv[mt][1] = ql ? c[3] : c[1];
    } else {
      sv[2 * mt][0] = c[0];
      sv[2 * mt][1] = c[1];
      sv[2 * mt + 1][0] = c[2];
      sv[2 * mt + 1][1] = c[3];
    }
  }
}

template <int HD, bool PACK>
struct RowState {
  float m[2], l[2];
  float o[Map<HD, PACK>::NC][2];
};

// One tile of Alg. 2 on the thread's score values: running max,
// alpha, SAS, row sum, per-row P scale and codes (to smem rows).
template <int HD, bool PACK, bool TAP, bool FULL, int BC, bool SF = false>
TA_DEV void softmax_tile(const DecodeArgs& a, RowState<HD, PACK>& st, int (&sv)[Map<HD, PACK>::NT * BC / 64][2], int nvalid,
                         const float (&cqk)[2], uint32_t pbuf, float lut_lane, float (&alpha)[2], float (&s_p)[2],
                         int (&sum_p)[2], bool tap, int tap_row, int g, int q) {
  using M = Map<HD, PACK>;
  constexpr int NT = M::NT * BC / 64;  // score values per thread and row
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int row = M::row(q, e);
    int smax = INT_MIN;
#pragma unroll
    for (int t = 0; t < NT; ++t)
      if (FULL || M::tok(t, g, q) < nvalid) smax = max(smax, sv[t][e]);
    smax = grp_maxi<PACK>(smax);
    const float m_prev = st.m[e];
    const float m_new = fmaxf(m_prev, __fmul_rn((float)smax, cqk[e]));
    // alpha = SAS(m_prev - m_new) (R-15); every lane evaluates (shuffle LUT)
    const float al_s = sas_eval_v<SF>(__fsub_rn(m_new, m_prev), lut_lane, a.sas.nr_abs);
    const float al = m_prev == -INFINITY ? 0.f : (a.alpha_mode == 1 && m_new == m_prev) ? 1.f : al_s;
    float pt[NT], rs = 0.f, pm = 0.f;
    const f32x2 m2 = pk2(m_new, m_new);
#pragma unroll
    for (int t = 0; t < NT; t += 2) {
      // x rounded on its own (scalar __fmul_rn: a packed multiply feeding the
      // subtraction would be contracted into an FFMA2)
      const f32x2 x2 = pk2(__fmul_rn((float)sv[t][e], cqk[e]), __fmul_rn((float)sv[t + 1][e], cqk[e]));
      const f32x2 p2 = sas_eval2_v<SF>(sub2(m2, x2), lut_lane, a.sas.nr_abs);  // R-13 / R-30
      float p0 = lo2(p2), p1 = hi2(p2);
      if (!FULL) {
        p0 = M::tok(t, g, q) < nvalid ? p0 : 0.f;
        p1 = M::tok(t + 1, g, q) < nvalid ? p1 : 0.f;
      }
      pt[t] = p0;
      pt[t + 1] = p1;
      rs += p0;
      rs += p1;
      pm = fmaxf(pm, fmaxf(p0, p1));
    }
    rs = grp_sumf<PACK>(rs);
    pm = grp_maxf<PACK>(pm);
    st.l[e] = al * st.l[e] + rs;
    st.m[e] = m_new;
    alpha[e] = al;
    // per-row P scale (Alg. 2, R-17)
    const float inv_p = pm > 0.f ? div_119_by(pm) : 0.f;
    s_p[e] = div_by_119(pm);
    // P codes rne(P~ 119 / max) (R-27): two per FFMA2 against 1.5 2^23; the low byte of each result's bits is
    // the code (stored as is) and the sum of the codes is the sum of the bits less NT x the magic's bits
    uint32_t spb = 0;
    const f32x2 ip2 = pk2(inv_p, inv_p), mg2 = pk2(kMagic, kMagic);
#pragma unroll
    for (int t = 0; t < NT; t += 2) {
      const f32x2 cb = fma2(pk2(pt[t], pt[t + 1]), ip2, mg2);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t bits = h ? (uint32_t)(cb >> 32) : (uint32_t)cb;
        spb += bits;
        sts_u8(pbuf + row * BC + M::tok(t + h, g, q), bits);
        if (TAP && tap && row == tap_row) {
          a.tap.p_codes[M::tok(t + h, g, q)] = (uint8_t)bits;
          a.tap.s_int[M::tok(t + h, g, q)] = M::tok(t + h, g, q) < nvalid ? sv[t + h][e] : 0;
        }
      }
    }
    sum_p[e] = grp_sumi<PACK>((int)(spb - (uint32_t)NT * kMagicBits));
    if (TAP && tap && row == tap_row && g == 0 && (!PACK || q < 2)) {
      a.tap.m_new[0] = m_new;
      a.tap.s_p[0] = s_p[e];
    }
  }
  __syncwarp();
}

// P V on a stage-2 block: raw V codes x P codes, then the exact per-channel
// fixup s_c * acc + z_c * sum(P) (Eq. 5 fold).  Buffer block: INT8 V, no fixup.
// B_c = 128: the two 64-token sub-blocks (layout.cuh) accumulate into the same
// IMMA sums before the fixup.
template <int HD, int BV, bool PACK, bool BUF, int BC>
TA_DEV void pv_block(uint32_t rec, const int8_t* vb, uint32_t pbuf, const int (&sum_p)[2],
                     int (&acc)[Map<HD, PACK>::NC][2], int g, int q) {
  const int rn = PACK ? (g & 3) : g;
  constexpr int NU = BC / kSub;     // 64-token sub-blocks
  constexpr int CB = kSub * BV / 8;  // bytes per channel of V codes per sub-block
  uint32_t bf[NU][2][2];
#pragma unroll
  for (int u = 0; u < NU; ++u)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      bf[u][j][0] = lds32(pbuf + rn * BC + kSub * u + 32 * j + 4 * q);
      bf[u][j][1] = lds32(pbuf + rn * BC + kSub * u + 32 * j + 16 + 4 * q);
    }
  const uint32_t codes = rec + 2 * HD;
  const bool ql = q >= 2;
#pragma unroll
  for (int mt = 0; mt < HD / 16; ++mt) {
    const int c0 = 16 * mt + g, c1 = c0 + 8;
    int c[4] = {0, 0, 0, 0};
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      // the channel pair's code words, loaded once for both units / k-steps
      uint32_t wv[4] = {0u, 0u, 0u, 0u};
      const uint32_t cu0 = codes + u * HD * CB;
      if (!BUF) {
        wv[0] = lds32(cu0 + c0 * CB + 4 * q);
        wv[1] = lds32(cu0 + c1 * CB + 4 * q);
        if (BV == 4) {
          wv[2] = lds32(cu0 + c0 * CB + 4 * (4 + q));
          wv[3] = lds32(cu0 + c1 * CB + 4 * (4 + q));
        }
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        uint32_t af[4];
        if (BUF) {
          const int8_t* vu = vb + kSub * u;
          af[0] = *reinterpret_cast<const uint32_t*>(vu + c0 * BC + 32 * j + 4 * q);
          af[1] = *reinterpret_cast<const uint32_t*>(vu + c1 * BC + 32 * j + 4 * q);
          af[2] = *reinterpret_cast<const uint32_t*>(vu + c0 * BC + 32 * j + 16 + 4 * q);
          af[3] = *reinterpret_cast<const uint32_t*>(vu + c1 * BC + 32 * j + 16 + 4 * q);
          const uint32_t b2[2] = {bf[u][j][0], bf[u][j][1]};
          imma_s8u8(c, af, b2);
        } else if (BV == 4) {
          // unit j: j = 0 low nibbles (tokens 4q+e | 32+4q+e), j = 1 high nibbles x16
          // (tokens 16+4q+e | 48+4q+e); word W = 4 j' + q holds both halves of k-step j'.
          const uint32_t mk = j ? 0xF0F0F0F0u : 0x0F0F0F0Fu;
#pragma unroll
          for (int i = 0; i < 4; ++i) af[i] = wv[i] & mk;
          // B rows of unit j: tokens (16 j + 4q..) and (32 + 16 j + 4q..)
          const uint32_t b2[2] = {j ? bf[u][0][1] : bf[u][0][0], j ? bf[u][1][1] : bf[u][1][0]};
          if (j == 0) {  // low nibbles: scale 1, accumulated in place
            imma_u8u8(c, af, b2);
          } else {
            int cu[4] = {0, 0, 0, 0};
            imma_u8u8(cu, af, b2);
#pragma unroll
            for (int i = 0; i < 4; ++i) c[i] += cu[i] >> 4;
          }
        } else {
          const int sh = 4 * j;
          af[0] = (wv[0] >> sh) & 0x03030303u;
          af[1] = (wv[1] >> sh) & 0x03030303u;
          af[2] = (wv[0] >> (sh + 2)) & 0x03030303u;
          af[3] = (wv[1] >> (sh + 2)) & 0x03030303u;
          const uint32_t b2[2] = {bf[u][j][0], bf[u][j][1]};
          imma_u8u8(c, af, b2);
        }
      }
    }
#pragma unroll
    for (int h = 0; h < (PACK ? 1 : 2); ++h) {
      const int hh = PACK ? (ql ? 1 : 0) : h;  // which channel of the pair (c0 / c1)
      const int ci = PACK ? mt : 2 * mt + h;
      const int ch = c0 + 8 * hh;
      // the channel's s_int / z_int, loaded once for both rows
      const int s_c = BUF ? 0 : (int)lds_u8(rec + ch), z_c = BUF ? 0 : lds_s8(rec + HD + ch);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        // selects, not c[2 * hh + e]: a runtime index would put c[] in local memory
        const int v = PACK ? (ql ? c[2 + e] : c[e]) : c[2 * h + e];
        acc[ci][e] = BUF ? v : s_c * v + z_c * sum_p[e];
      }
    }
  }
}

// Units of work of sequence b for one kv head: the blocks of [blk_begin,
// blk_end) it has flushed, plus the INT8 buffer block when it is used.
struct SeqUnits {
  int jb, nblk, nbuf, units;
};
TA_DEV SeqUnits seq_units(const DecodeArgs& a, int b) {
  const int nb = a.counters[2 * b], nbuf = a.counters[2 * b + 1];
  const int jb = min(a.blk_begin, nb), je = a.blk_end < 0 ? nb : min(a.blk_end, nb);
  const int nblk = max(0, je - jb);
  return SeqUnits{jb, nblk, nbuf, nblk + ((a.with_buffer && nbuf > 0) ? 1 : 0)};
}

// One online-softmax pass of Alg. 2 for (b, kv head) over the
// blocks [j0, j1) and, if use_buf, the buffer block last; writes the
// normalised partial (O, L) of the G query rows to part `part` (rows
// part*G .. part*G+G-1 of o_parts / lse_parts; the final [B][Hq] layout when
// part == b*Hkv + kvh).  `it` counts the ring iterations of this warp across
// segments (stage = it & 1, mbarrier parity = (it >> 1) & 1).
template <int HD, bool PACK, bool TAP, int BC, bool SF>
TA_DEV void decode_segment(const DecodeArgs& a, DecodeSmem<HD, PACK, BC>& sm, int b, int kvh, int j0, int j1, bool use_buf,
                           int nbuf, size_t part, bool tap_ok, uint32_t& it, int lane) {
  using M = Map<HD, PACK>;
  const int g = lane >> 2, q = lane & 3;
  const int G = a.G;
  const int kvr = kvh / a.RG;  // the real KV head of this (virtual) head
  const int bitsK = a.bits[kvr * 2], bitsV = a.bits[kvr * 2 + 1];
  const size_t slotK = ((size_t)b * (a.Hkv / a.RG) + kvr) * 2, slotV = slotK + 1;
  constexpr int REC = rec_bytes(HD, BC);
  constexpr int NT = M::NT * BC / 64;
  const uint32_t bytesK = 2 * HD + BC * HD * bitsK / 8, bytesV = 2 * HD + BC * HD * bitsV / 8;
  const float lut_lane = sas_lut_lane(a.sas, lane);
  const int tap_row = TAP && tap_ok && a.tap.batch == b && a.tap.head / G == kvh ? a.tap.head % G : -1;
  const uint32_t pbuf = smem_u32(&sm.p[0][0]), q1s = smem_u32(&sm.q1[0][0]);

  __syncwarp();
  const uint32_t it0 = it;
  auto issue = [&](int j, int stg) {
    if (lane == 0) {
      mbar_expect_tx(&sm.bar[stg], bytesK + bytesV);
      bulk_load(sm.rec[stg][0], a.block_rec + (slotK * a.max_blocks + j) * REC, bytesK, &sm.bar[stg]);
      bulk_load(sm.rec[stg][1], a.block_rec + (slotV * a.max_blocks + j) * REC, bytesV, &sm.bar[stg]);
    }
  };
  if (j0 < j1) issue(j0, it0 & 1);
  if (j0 + 1 < j1) issue(j0 + 1, (it0 + 1) & 1);

  // q stage-1 quantisation per (b, head) vector (Alg. 2): lane quad g
  // quantises row g (rows >= G are zero).
  float s_q_row = 0.f;
  {
    constexpr int R = HD / 4;
    float qa = 0.f;
    float xv[R];
    const __half* qp = a.q + ((size_t)b * a.Hq + kvh * G + g) * HD + q * R;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      xv[i] = g < G ? __half2float(qp[i]) : 0.f;
      qa = fmaxf(qa, fabsf(xv[i]));
    }
    qa = fmaxf(qa, __shfl_xor_sync(0xffffffffu, qa, 1));
    qa = fmaxf(qa, __shfl_xor_sync(0xffffffffu, qa, 2));
    const float inv = qa > 0.f ? div_119_by(qa) : 0.f;
    s_q_row = st1_scale(div_by_119(qa), a.scale_fp16);  // (FP16 variant: R-29)
#pragma unroll
    for (int i = 0; i < R; i += 4)
      if (g < (PACK ? 4 : 8))  // rows >= G are zero (and absent on the packed path)
        *reinterpret_cast<uint32_t*>(&sm.q1[g][q * R + i]) =
          pack4_lo(rint_prod_bits(xv[i], inv), rint_prod_bits(xv[i + 1], inv), rint_prod_bits(xv[i + 2], inv),
                   rint_prod_bits(xv[i + 3], inv));
    if (TAP && g == tap_row) {
      for (int i = 0; i < R; ++i) a.tap.q1[q * R + i] = sm.q1[g][q * R + i];
      if (q == 0) a.tap.s_q[0] = s_q_row;
    }
  }
  __syncwarp();
  // The lane's K-channel region of its B-fragment row: row g (general) or row
  // g & 3 (packed), as packed bytes (dp4a) and as ints (products).
  const int brow = PACK ? (g & 3) : g;
  uint4 q1r[HD / 64];
  int qv[HD / 4];
#pragma unroll
  for (int i = 0; i < HD / 64; ++i) {
    q1r[i] = lds128(q1s + brow * HD + q * (HD / 4) + 16 * i);
#pragma unroll
    for (int e = 0; e < 16; ++e) qv[16 * i + e] = (int)(byte_of(q1r[i], e) << (8 * (e & 3)));  // byte-positioned
  }
  const int rq = PACK ? (q & 1) : q;
  const float sq2[2] = {__shfl_sync(0xffffffffu, s_q_row, 8 * rq), __shfl_sync(0xffffffffu, s_q_row, 8 * rq + 4)};

  RowState<HD, PACK> st;
  st.m[0] = st.m[1] = -INFINITY;
  st.l[0] = st.l[1] = 0.f;
#pragma unroll
  for (int c = 0; c < M::NC; ++c) st.o[c][0] = st.o[c][1] = 0.f;

  auto update = [&](const int (&acc)[M::NC][2], const float (&alpha)[2], const float (&cpv)[2], bool tap) {
    // o = alpha o + cpv acc for the lane's two rows at once (FMUL2 then FFMA2: the same two roundings)
    const f32x2 al2 = pk2(alpha[0], alpha[1]), cp2 = pk2(cpv[0], cpv[1]);
#pragma unroll
    for (int c = 0; c < M::NC; ++c) {
      const f32x2 o2 = fma2(al2, pk2(st.o[c][0], st.o[c][1]), mul2(cp2, pk2((float)acc[c][0], (float)acc[c][1])));
      st.o[c][0] = lo2(o2);
      st.o[c][1] = hi2(o2);
#pragma unroll
      for (int e = 0; e < 2; ++e)
        if (TAP && tap && M::row(q, e) == tap_row) a.tap.pv_int[M::chan(c, g, q)] = acc[c][e];
    }
  };

  for (int j = j0; j < j1; ++j) {
    const uint32_t itj = it0 + (uint32_t)(j - j0);
    const int stg = itj & 1;
    mbar_wait(&sm.bar[stg], (itj >> 1) & 1);
    const uint32_t recK = smem_u32(sm.rec[stg][0]), recV = smem_u32(sm.rec[stg][1]);
    int sv[NT][2];
    if (bitsK == 4) qk_block<HD, 4, PACK, BC>(recK, qv, q1r, sv, g, q);
    else qk_block<HD, 2, PACK, BC>(recK, qv, q1r, sv, g, q);
    const float sK = a.s_parent[slotK * a.max_blocks + j], sV = a.s_parent[slotV * a.max_blocks + j];
    const float cqk[2] = {__fmul_rn(__fmul_rn(sq2[0], sK), a.scale), __fmul_rn(__fmul_rn(sq2[1], sK), a.scale)};
    const bool tap = TAP && tap_row >= 0 && a.tap.j_block == j;
    float alpha[2], s_p[2];
    int sum_p[2];
    softmax_tile<HD, PACK, TAP, true, BC, SF>(a, st, sv, BC, cqk, pbuf, lut_lane, alpha, s_p, sum_p, tap, tap_row, g, q);
    int acc[M::NC][2];
    if (bitsV == 4) pv_block<HD, 4, PACK, false, BC>(recV, nullptr, pbuf, sum_p, acc, g, q);
    else pv_block<HD, 2, PACK, false, BC>(recV, nullptr, pbuf, sum_p, acc, g, q);
    const float cpv[2] = {__fmul_rn(s_p[0], sV), __fmul_rn(s_p[1], sV)};
    update(acc, alpha, cpv, tap);
    __syncwarp();
    if (j + 2 < j1) issue(j + 2, stg);
  }

  it = it0 + (uint32_t)max(0, j1 - j0);

  if (use_buf) {
    // Buffer block (INT8, universal scale, n_buf valid keys), last.
    const int8_t* kb = a.buf + slotK * (size_t)(BC * HD);
    const int8_t* vb = a.buf + slotV * (size_t)(BC * HD);
    const float sK = st1_scale(div_by_119(a.a_univ[slotK]), a.scale_fp16),
                sV = st1_scale(div_by_119(a.a_univ[slotV]), a.scale_fp16);
    int sv[NT][2];
    qk_buffer<HD, PACK, BC>(kb, q1s, sv, g, q);
    const float cqk[2] = {__fmul_rn(__fmul_rn(sq2[0], sK), a.scale), __fmul_rn(__fmul_rn(sq2[1], sK), a.scale)};
    const bool tap = TAP && tap_row >= 0 && a.tap.j_block == -1;
    float alpha[2], s_p[2];
    int sum_p[2];
    softmax_tile<HD, PACK, TAP, false, BC, SF>(a, st, sv, nbuf, cqk, pbuf, lut_lane, alpha, s_p, sum_p, tap, tap_row, g,
                                              q);
    int acc[M::NC][2];
    pv_block<HD, 4, PACK, true, BC>(0, vb, pbuf, sum_p, acc, g, q);
    const float cpv[2] = {__fmul_rn(s_p[0], sV), __fmul_rn(s_p[1], sV)};
    update(acc, alpha, cpv, tap);
  }

  // O = diag(l)^-1 O, L = m + log l; empty -> O = 0, L = -inf.
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int row = M::row(q, e);
    if (row >= G) continue;
    const bool empty = st.l[e] == 0.f;
    const float inv_l = empty ? 0.f : 1.f / st.l[e];
    const size_t orow = (size_t)b * a.Hq + kvh * G + row;
    const size_t prow = part * G + row;
    const size_t base = prow * HD;
#pragma unroll
    for (int c = 0; c < M::NC; ++c) {
      const float v = st.o[c][e] * inv_l;
      const int ch = M::chan(c, g, q);
      if (a.o_parts) a.o_parts[base + ch] = v;
      if (a.o16) a.o16[orow * HD + ch] = __float2half_rn(v);
    }
    if (g == 0 && (!PACK || q < 2))
      a.lse_parts[prow] = empty ? -INFINITY : st.m[e] + logf(st.l[e]);
  }
}


// Two schedules:
//  * n_splits >= 1: one warp per (b, kv head, split), the split cutting the
//    block range into n_splits contiguous ranges of ceil(n / n_splits) blocks
//    (buffer with the last); part = split * B * Hkv + b * Hkv + kvh.
//  * balanced (n_splits == 0): a persistent grid of W warps; the units of all
//    (b, kv head) in b-major, kv-head, block order (buffer last) are cut into
//    W contiguous chunks of C = max(kMinUnits, ceil(total / W)) units; a warp
//    runs one pass per (b, kv head) piece of its chunk; piece (bh, w) writes
//    part bh + w (unique: pieces of a later bh belong to no earlier warp).
template <int HD, bool PACK, bool TAP, int BC, bool SF>
__global__ void __launch_bounds__(32 * kWarpsPerCta) decode_kernel(const __grid_constant__ DecodeArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  DecodeSmem<HD, PACK, BC>& sm = reinterpret_cast<DecodeSmem<HD, PACK, BC>*>(smem_raw)[warp];
  pdl_trigger();  // the combine grid may launch once every decode CTA has started
  pdl_wait();     // (launched with PDL after the append kernels: their counters / buffer)
  if (lane == 0) {
    mbar_init(&sm.bar[0], 1);
    mbar_init(&sm.bar[1], 1);
    fence_barrier_init();
  }
  __syncwarp();
  uint32_t it = 0;
  if (a.n_splits > 0) {
    const int task = blockIdx.x * kWarpsPerCta + warp;
    if (task >= a.B * a.Hkv * a.n_splits) return;
    const int split = task % a.n_splits, bh = task / a.n_splits, b = bh / a.Hkv, kvh = bh % a.Hkv;
    const SeqUnits su = seq_units(a, b);
    const int je = su.jb + su.nblk, per = (su.nblk + a.n_splits - 1) / a.n_splits;
    const int j0 = min(su.jb + split * per, je), j1 = min(j0 + per, je);
    const bool use_buf = a.with_buffer && split == a.n_splits - 1 && su.nbuf > 0;
    decode_segment<HD, PACK, TAP, BC, SF>(a, sm, b, kvh, j0, j1, use_buf, su.nbuf, (size_t)split * a.B * a.Hkv + bh,
                                  split == 0, it, lane);
    return;
  }
  // balanced schedule
  const int W = gridDim.x * kWarpsPerCta, w = blockIdx.x * kWarpsPerCta + warp;
  int tot = 0;
  for (int b0 = 0; b0 < a.B; b0 += 32)
    if (b0 + lane < a.B) tot += seq_units(a, b0 + lane).units;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  tot *= a.Hkv;
  const int C = max(kMinUnits, (tot + W - 1) / W);
  int pos = w * C;
  const int end = min(pos + C, tot);
  if (pos >= end) return;
  // locate the sequence holding unit `pos`: lane-parallel scan over b (a
  // serial walk would chain B dependent global loads before the first block)
  int b = 0, base = 0;
  for (int b0 = 0, carry = 0; b0 < a.B; b0 += 32) {
    const int u = b0 + lane < a.B ? seq_units(a, b0 + lane).units * a.Hkv : 0;
    int incl = u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const unsigned hit = __ballot_sync(0xffffffffu, carry + incl > pos);
    if (hit) {
      const int l = __ffs(hit) - 1;
      b = b0 + l;
      base = carry + __shfl_sync(0xffffffffu, incl - u, l);
      break;
    }
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  SeqUnits su = seq_units(a, b);
  while (pos < end) {
    const int U = su.units, kvh = (pos - base) / U, u0 = (pos - base) % U;
    const int seg_end = min(end, base + (kvh + 1) * U), u1 = seg_end - (base + kvh * U);
    decode_segment<HD, PACK, TAP, BC, SF>(a, sm, b, kvh, su.jb + u0, su.jb + min(u1, su.nblk), u1 > su.nblk, su.nbuf,
                                  (size_t)b * a.Hkv + kvh + w, true, it, lane);
    pos = seg_end;
    while (pos < end && pos >= base + su.units * a.Hkv) {
      base += su.units * a.Hkv;
      su = seq_units(a, ++b);
    }
  }
}

// Log-sum-exp merge of n partial (O_s, L_s) of one output row (R-23):
// L = max + log sum_s e^{L_s - max},  O = sum_s (e^{L_s - max} / wsum) O_s.
// Part s sits at lse[s * lse_stride], o[s * o_stride + c].  W = blockDim / 32
// <= kCombWarps warps (comb_warps: about 4 parts per warp): warp 0 computes the
// weights into shared memory (lane-strided sums, fixed butterfly order); warp k
// then sums the contiguous part range [k n / W, (k+1) n / W) in ascending order for all d channels (d / 32
// consecutive channels per lane, one vector load per part, 8 parts in flight),
// and the W partial rows are added in warp order -- deterministic, and with
// many parts in flight per row instead of one serial chain (B = 1 decode runs
// 32 rows of 128-512 parts: up to 16 warps, 8 parts each in one round of loads).
constexpr int kCombWarps = 16;
// about 4 parts per warp up to 8 warps; 16 warps (8 parts each) from 128 parts on (measured: 8 warps are
// 2 % faster at 64 parts per row and 2560 rows, 16 warps 9 % faster at 256 parts and 32 rows)
static inline int comb_warps(int n) { return n >= 128 ? 16 : n >= 32 ? 8 : std::max(1, (n + 3) / 4); }
template <int VEC>
TA_DEV void combine_row(int n, const float* __restrict__ lse, size_t lse_stride, const float* __restrict__ o,
                        size_t o_stride, int d, float* w, float (*part)[128], __half* o16, float* o32, float* L_out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (warp == 0) {
    float lmax = -INFINITY;
    for (int s = lane; s < n; s += 32) lmax = fmaxf(lmax, lse[s * lse_stride]);
#pragma unroll
    for (int x = 16; x > 0; x >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, x));
    float wsum = 0.f;
    if (lmax != -INFINITY)
      for (int s = lane; s < n; s += 32) {
        const float e = expf(lse[s * lse_stride] - lmax);
        w[s] = e;
        wsum += e;
      }
#pragma unroll
    for (int x = 16; x > 0; x >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, x);
    const float inv = lmax != -INFINITY ? 1.f / wsum : 0.f;
    __syncwarp();
    for (int s = lane; s < n; s += 32) w[s] = lmax != -INFINITY ? w[s] * inv : 0.f;
    if (lane == 0) {
      w[n] = lmax;
      if (L_out) *L_out = lmax != -INFINITY ? lmax + logf(wsum) : -INFINITY;
    }
  }
  __syncthreads();
  const bool live = w[n] != -INFINITY;
  const int c0 = lane * VEC;
  float acc[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) acc[v] = 0.f;
  if (live && c0 < d) {
    const int s0 = (int)((long long)warp * n / nw), s1 = (int)((long long)(warp + 1) * n / nw);
    int s = s0;
    for (; s + 8 <= s1; s += 8) {
      float x[8][VEC];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float* src = o + (size_t)(s + k) * o_stride + c0;
        if (VEC == 4) {
          const float4 t = *reinterpret_cast<const float4*>(src);
          x[k][0] = t.x; x[k][VEC > 1 ? 1 : 0] = t.y; x[k][VEC > 2 ? 2 : 0] = t.z; x[k][VEC > 3 ? 3 : 0] = t.w;
        } else if (VEC == 2) {
          const float2 t = *reinterpret_cast<const float2*>(src);
          x[k][0] = t.x; x[k][VEC > 1 ? 1 : 0] = t.y;
        } else {
#pragma unroll
          for (int v = 0; v < VEC; ++v) x[k][v] = src[v];
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[v] += w[s + k] * x[k][v];
    }
    for (; s < s1; ++s)
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[v] += w[s] * o[(size_t)s * o_stride + c0 + v];
  }
  if (c0 < d)
#pragma unroll
    for (int v = 0; v < VEC; ++v) part[warp][c0 + v] = acc[v];
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float out = 0.f;
#pragma unroll
    for (int k = 0; k < kCombWarps; ++k)
      if (k < nw) out += part[k][c];
    if (o16) o16[c] = __float2half_rn(out);
    if (o32) o32[c] = out;
  }
}

// Balanced schedule (R-23): one CTA per output row (b, h); the pieces of
// (b, kv head) are the parts bh + w for the warps w whose chunks meet its unit
// range.
template <int VEC>
__global__ void __launch_bounds__(32 * kCombWarps) combine_balanced_kernel(const __grid_constant__ DecodeArgs a, int W,
                                                                             int d) {
  extern __shared__ float w[];  // [n + 1]
  __shared__ float part[kCombWarps][128];
  pdl_wait();  // the decode grid's partials
  const int r = blockIdx.x, b = r / a.Hq, h = r % a.Hq, kvh = h / a.G, row = h % a.G, lane = threadIdx.x & 31;
  int tot = 0, before = 0;
  for (int b0 = 0; b0 < a.B; b0 += 32) {
    const int bb = b0 + lane;
    const int u = bb < a.B ? seq_units(a, bb).units : 0;
    tot += u;
    before += bb < b ? u : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    tot += __shfl_xor_sync(0xffffffffu, tot, o);
    before += __shfl_xor_sync(0xffffffffu, before, o);
  }
  const int U = seq_units(a, b).units;
  const int C = max(kMinUnits, (tot * a.Hkv + W - 1) / W);
  const int start = before * a.Hkv + kvh * U;
  const int bh = b * a.Hkv + kvh;
  const int w0 = U > 0 ? start / C : 0, n = U > 0 ? (start + U - 1) / C - w0 + 1 : 0;
  const size_t p0 = (size_t)(bh + w0) * a.G + row;
  combine_row<VEC>(n, a.lse_parts + p0, a.G, a.o_parts + p0 * d, (size_t)a.G * d, d, w, part,
                   a.fin_o16 ? a.fin_o16 + (size_t)r * d : nullptr, a.fin_o32 ? a.fin_o32 + (size_t)r * d : nullptr,
                   threadIdx.x == 0 ? a.fin_lse + r : nullptr);
}

// Equal splits / turbo_combine_lse: one CTA per row r, parts s at
// lse_parts[s rows + r], o_parts[(s rows + r) d + c].
template <int VEC>
__global__ void __launch_bounds__(32 * kCombWarps) combine_kernel(int n_parts, int rows, int d,
                                                                    const float* __restrict__ o_parts,
                                                                    const float* __restrict__ lse_parts,
                                                                    __half* __restrict__ o16, float* __restrict__ o32,
                                                                    float* __restrict__ lse) {
  extern __shared__ float w[];  // [n_parts + 1]
  __shared__ float part[kCombWarps][128];
  pdl_wait();  // the decode grid's partials
  const int r = blockIdx.x;
  combine_row<VEC>(n_parts, lse_parts + r, rows, o_parts + (size_t)r * d, (size_t)rows * d, d, w, part,
                   o16 ? o16 + (size_t)r * d : nullptr, o32 ? o32 + (size_t)r * d : nullptr,
                   threadIdx.x == 0 ? lse + r : nullptr);
}

static void launch_combine_kernel(int n_parts, int rows, int d, const float* o_parts, const float* lse_parts,
                                  __half* o16, float* o32, float* lse, cudaStream_t st) {
  // (n_parts + 1) weights: up to 48 KB at the 12000-part bound, over the default 48 KB
  // dynamic limit once the 4 KB of static shared memory are added -- raise it explicitly.
  const size_t smem = (n_parts + 1) * sizeof(float);
  const int thr = 32 * comb_warps(n_parts);
  if (d == 128) {
    cudaFuncSetAttribute(combine_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    ta_host::launch_pdl(combine_kernel<4>, dim3(rows), dim3(thr), smem, st, n_parts, rows, d, o_parts, lse_parts, o16,
                        o32, lse);
  } else {
    cudaFuncSetAttribute(combine_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    ta_host::launch_pdl(combine_kernel<2>, dim3(rows), dim3(thr), smem, st, n_parts, rows, d, o_parts, lse_parts, o16,
                        o32, lse);
  }
}

}  // namespace ta

namespace ta_host {
using namespace ta;

template <int HD, bool PK, bool TP>
static int decode_ctas_per_sm() {
  int n = 0;
  const size_t smem = sizeof(DecodeSmem<HD, PK, 64>) * kWarpsPerCta;
  cudaFuncSetAttribute(decode_kernel<HD, PK, TP, 64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, decode_kernel<HD, PK, TP, 64, false>, 32 * kWarpsPerCta, smem) !=
      cudaSuccess)
    n = 0;
  return n;
}

// Worker warps of the balanced schedule on the current device: every SM
// filled to the decode kernel's occupancy (of the B_c = 64 kernel; with B_c = 128
// the same count is a plain partition of the units).
int decode_workers(int Hq, int Hkv, int HD) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return 0;
  const bool pack = Hkv > 0 && Hq / Hkv <= 4;
  const int per_sm = HD == 128 ? (pack ? decode_ctas_per_sm<128, true, false>() : decode_ctas_per_sm<128, false, false>())
                               : (pack ? decode_ctas_per_sm<64, true, false>() : decode_ctas_per_sm<64, false, false>());
  return sms * per_sm * kWarpsPerCta;
}

// Row groups per KV head: the least RG with G / RG <= 8 rows that divides G (G <= 8: 1).
int decode_row_groups(int G) {
  for (int r = (G + 7) / 8; r <= G; ++r)
    if (G % r == 0) return r;
  return G;
}

size_t decode_workspace(int B, int Hq, int Hkv, int HD, int S) {
  if (S == 1) return 0;
  if (S > 1) return (size_t)S * B * Hq * (HD + 1) * sizeof(float);
  // balanced: parts bh + w < B * Hkv' + W (Hkv' = Hkv x row groups), G' rows of d + 1 floats each
  // (S < 0: W = -S workers)
  const int RG = decode_row_groups(Hq / Hkv), Hv = Hkv * RG;
  const int W = S < 0 ? -S : decode_workers(Hq, Hv, HD);
  return W <= 0 ? 0 : ((size_t)B * Hv + W) * (Hq / Hv) * (HD + 1) * sizeof(float);
}

cudaError_t launch_decode(const turbo_params_t* p, const turbo_kv_cache_t* c, int Hq, const __half* q, int blk_begin,
                          int blk_end, int with_buffer, int S, void* ws, __half* o, float* o_part, float* lse,
                          cudaStream_t st) {
  const int RG = decode_row_groups(Hq / c->n_kv_heads);
  const int B = c->batch, H = c->n_kv_heads * RG, HD = c->head_dim;  // H: virtual KV heads (G > 8)
  DecodeArgs a;
  memset(&a, 0, sizeof(a));
  a.RG = RG;
  a.q = q;
  a.block_rec = c->block_rec;
  a.s_parent = c->s_parent;
  a.buf = c->buf;
  a.a_univ = c->a_univ;
  a.counters = c->counters;
  a.bits = c->bits_dev;
  a.B = B;
  a.Hq = Hq;
  a.Hkv = H;
  a.G = Hq / H;
  a.max_blocks = c->max_blocks;
  a.blk_begin = blk_begin;
  a.blk_end = blk_end;
  a.with_buffer = with_buffer;
  a.n_splits = S;
  a.alpha_mode = p->alpha_mode;
  a.scale_fp16 = p->scale_fp16;
  a.sas_fp16 = p->sas_fp16;
  a.scale = p->softmax_scale;
  fill_sas_const(&a.sas, p->sas_nr);
  const bool has_tap = p->debug_tap != nullptr;
  if (has_tap) a.tap = *reinterpret_cast<const turbo_debug_tap_t*>(p->debug_tap);
  const int W = S == 0 ? decode_workers(Hq, H, HD) : S < 0 ? -S : 0;  // balanced: device or explicit workers
  if (S <= 0 && W <= 0) return cudaErrorInvalidConfiguration;
  if (S == 1) {
    a.o_parts = o_part;
    a.lse_parts = lse;
    a.o16 = o;
  } else {
    const size_t parts = S > 1 ? (size_t)S * B * H : (size_t)B * H + W;
    a.o_parts = reinterpret_cast<float*>(ws);
    a.lse_parts = a.o_parts + parts * a.G * HD;
    a.fin_o16 = o;
    a.fin_o32 = o_part;
    a.fin_lse = lse;
  }
  const int tasks = S > 0 ? B * H * S : W;
  const dim3 grid((tasks + kWarpsPerCta - 1) / kWarpsPerCta);
  const bool pack = a.G <= 4;
#define TA_DEC_S(HDV, PK, TP, BCV, SFV)                                                                   \
  {                                                                                                         \
    const size_t smem = sizeof(DecodeSmem<HDV, PK, BCV>) * kWarpsPerCta;                                    \
    cudaFuncSetAttribute(decode_kernel<HDV, PK, TP, BCV, SFV>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                         (int)smem);                                                                        \
    launch_pdl(decode_kernel<HDV, PK, TP, BCV, SFV>, grid, dim3(32 * kWarpsPerCta), smem, st, a);           \
  }
#define TA_DEC_B(HDV, PK, TP, BCV) \
  if (a.sas_fp16) TA_DEC_S(HDV, PK, TP, BCV, true) else TA_DEC_S(HDV, PK, TP, BCV, false)
#define TA_DEC(HDV, PK, TP) \
  if (c->block_kv == 64) TA_DEC_B(HDV, PK, TP, 64) else TA_DEC_B(HDV, PK, TP, 128)
#define TA_DEC2(HDV)                                                  \
  if (pack) {                                                         \
    if (has_tap) TA_DEC(HDV, true, true) else TA_DEC(HDV, true, false)  \
  } else {                                                            \
    if (has_tap) TA_DEC(HDV, false, true) else TA_DEC(HDV, false, false) \
  }
  if (HD == 128) {
    TA_DEC2(128)
  } else {
    TA_DEC2(64)
  }
#undef TA_DEC2
#undef TA_DEC
#undef TA_DEC_B
#undef TA_DEC_S
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || S == 1) return e;
  if (S <= 0) {
    const size_t smem = (size_t)(W + 2) * sizeof(float);  // a row's pieces: at most W
    // pieces per row ~ W / (B Hkv) + 1
    const int thr = 32 * comb_warps(W / (B * H) + 1);
    if (HD == 128) {
      cudaFuncSetAttribute(combine_balanced_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      launch_pdl(combine_balanced_kernel<4>, dim3(B * Hq), dim3(thr), smem, st, a, W, HD);
    } else {
      cudaFuncSetAttribute(combine_balanced_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      launch_pdl(combine_balanced_kernel<2>, dim3(B * Hq), dim3(thr), smem, st, a, W, HD);
    }
  } else {
    const int rows = B * Hq;
    launch_combine_kernel(S, rows, HD, a.o_parts, a.lse_parts, o, o_part, lse, st);
  }
  return cudaGetLastError();
}

cudaError_t launch_combine(int n_parts, int rows, int d, const float* o_parts, const float* lse_parts, __half* o,
                           float* o32, float* lse, cudaStream_t st) {
  launch_combine_kernel(n_parts, rows, d, o_parts, lse_parts, o, o32, lse, st);
  return cudaGetLastError();
}
}  // namespace ta_host
