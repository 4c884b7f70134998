// decode.cu -- Algorithm 2 (TurboAttention decode) on sm_100a,
// plus the split-KV log-sum-exp combine (R-23).
//
// One WARP = one (batch, kv head, split) task; it owns the G = Hq/Hkv query
// rows of that KV head (GQA, R-22) and walks its contiguous block range in
// Alg. 2 order.  Block records (s_int | z_int | packed codes) stream through a
// per-warp 2-stage smem ring with cp.async.bulk (TMA 1-D) + mbarrier; codes are
// unpacked in registers straight into mma.sync m16n8k32 IMMA fragments.
//
// Integer dequantisation (Alg. 2) is folded exactly (Eq. 5, P:275-283,
// linear because reconstructions never clamp, R-6):
//   S[t]    = sum_c q1_c (code_tc s_c + z_c)
//           = 128 * sum_c hi(q1_c s_c) code_tc + sum_c lo(q1_c s_c) code_tc + sum_c q1_c z_c
//   PV[c]   = sum_t P_t (code_tc s_c + z_c) = s_c * sum_t P_t code_tc + z_c * sum_t P_t
// with q1_c s_c = 128 hi + lo, hi in [-75, 74] (s8), lo in [0, 127] (u8), so the
// tensor cores see only raw 4-bit / 2-bit codes.
#include <climits>
#include <cstring>

#include "common.cuh"
#include "layout.cuh"

namespace ta {

constexpr int kWarpsPerCta = 4;

template <int HD>
struct DecodeWarpSmem {
  uint8_t rec[2][2][rec_bytes(HD)];  // [stage][K,V][record]
  int8_t q1[8][HD];
  uint8_t p[8][kBc];
  uint64_t bar[2];
};

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
  int B, Hq, Hkv, G, max_blocks, blk_begin, blk_end, with_buffer, n_splits, alpha_mode;
  float scale;
  SasConst sas;
  int has_tap;
  turbo_debug_tap_t tap;
};

TA_DEV uint32_t byte_of(const uint4& v, int i) {
  const uint32_t w = i < 4 ? v.x : i < 8 ? v.y : i < 12 ? v.z : v.w;
  return (w >> (8 * (i & 3))) & 0xFFu;
}
TA_DEV int sbyte_of(const uint4& v, int i) { return (int)(int8_t)(uint8_t)byte_of(v, i); }

TA_DEV int shfl_max_g(int v) {
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
TA_DEV float shfl_maxf_g(float v) {
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
TA_DEV float shfl_sumf_g(float v) {
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
TA_DEV int shfl_sum_g(int v) {
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Channel of the low k-slot m (0..3) of k-step j for lane quad q (layout.cuh):
// the high slot is the next channel.
template <int HD, int BITS>
TA_DEV constexpr int k_chan(int q, int j, int m) {
  return BITS == 4 ? q * (HD / 4) + 8 * j + 2 * m : q * (HD / 4) + 16 * (j >> 1) + 4 * m + 2 * (j & 1);
}

// Per-warp online-softmax state of the thread's two rows (2q, 2q+1) and its
// O slice (channels 16 mt + g and 16 mt + g + 8, mt < HD/16).
template <int HD>
struct RowState {
  float m[2], l[2];
  float o[HD / 16][4];
};

// One tile (64 keys) of Alg. 2 given S_int in C-fragment order.
// s[mt][i]: token 16mt + g (+8 for i >= 2), row 2q + (i & 1).
template <int HD>
TA_DEV void softmax_tile(const DecodeArgs& a, RowState<HD>& st, int (&s)[4][4], int nvalid, const float (&cqk)[2],
                         uint8_t (*pbuf)[kBc], float lut_lane, float (&alpha)[2], float (&s_p)[2], int (&sum_p)[2],
                         bool tap, int tap_row, int g, int q) {
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    int smax = INT_MIN;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      if (16 * mt + g < nvalid) smax = max(smax, s[mt][e]);
      if (16 * mt + g + 8 < nvalid) smax = max(smax, s[mt][2 + e]);
    }
    smax = shfl_max_g(smax);
    const float m_prev = st.m[e];
    const float m_new = fmaxf(m_prev, __fmul_rn((float)smax, cqk[e]));
    // alpha = SAS(m_prev - m_new) (R-15); evaluated by every lane (shuffle LUT)
    const float al_s = sas_eval(__fsub_rn(m_new, m_prev), lut_lane, a.sas.nr_abs);
    const float al = m_prev == -INFINITY ? 0.f : (a.alpha_mode == 1 && m_new == m_prev) ? 1.f : al_s;
    float pt[8], rs = 0.f, pm = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int mt = i >> 1, hi = i & 1, tok = 16 * mt + g + 8 * hi;
      const float x = __fmul_rn((float)s[mt][2 * hi + e], cqk[e]);
      float p = sas_eval(__fsub_rn(m_new, x), lut_lane, a.sas.nr_abs);
      p = tok < nvalid ? p : 0.f;
      pt[i] = p;
      rs += p;
      pm = fmaxf(pm, p);
    }
    rs = shfl_sumf_g(rs);
    pm = shfl_maxf_g(pm);
    st.l[e] = al * st.l[e] + rs;
    st.m[e] = m_new;
    alpha[e] = al;
    // per-row P scale (Alg. 2, R-17)
    const float inv_p = pm > 0.f ? __fdiv_rn(kDiv, pm) : 0.f;
    s_p[e] = __fdiv_rn(pm, kDiv);
    int sp = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int mt = i >> 1, hi = i & 1, tok = 16 * mt + g + 8 * hi;
      const int c = rint_prod(pt[i], inv_p);
      sp += c;
      pbuf[2 * q + e][tok] = (uint8_t)c;
      if (tap && 2 * q + e == tap_row) a.tap.p_codes[tok] = (uint8_t)c;
    }
    sum_p[e] = shfl_sum_g(sp);
    if (tap && 2 * q + e == tap_row && g == 0) {
      a.tap.m_new[0] = m_new;
      a.tap.s_p[0] = s_p[e];
    }
  }
  __syncwarp();
}

template <int HD>
TA_DEV void pv_update(RowState<HD>& st, const int (&acc)[HD / 16][4], const float (&alpha)[2], const float (&cpv)[2]) {
#pragma unroll
  for (int mt = 0; mt < HD / 16; ++mt)
#pragma unroll
    for (int i = 0; i < 4; ++i) st.o[mt][i] = __fmaf_rn(alpha[i & 1], st.o[mt][i], cpv[i & 1] * (float)acc[mt][i]);
}

template <int HD, int BK>
TA_DEV void qk_q2(const uint8_t* rec, const uint4 (&q1r)[HD / 64], int (&s)[4][4], int g, int q) {
  // B fragments: hi/lo split of q1_c * s_c over the lane's channel region.
  const int R = HD / 4;
  uint4 sv[HD / 64];
#pragma unroll
  for (int i = 0; i < HD / 64; ++i) sv[i] = *reinterpret_cast<const uint4*>(rec + q * R + 16 * i);
  constexpr int KS = HD / 32;
  uint32_t bhi[KS][2], blo[KS][2];
#pragma unroll
  for (int j = 0; j < KS; ++j)
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      uint32_t vh = 0, vl = 0;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int loc = k_chan<HD, BK>(0, j, m) + h2;  // channel offset inside the region
        const int prod = sbyte_of(q1r[loc >> 4], loc & 15) * (int)byte_of(sv[loc >> 4], loc & 15);
        vh |= (uint32_t)((prod >> 7) & 0xFF) << (8 * m);
        vl |= (uint32_t)(prod & 0x7F) << (8 * m);
      }
      bhi[j][h2] = vh;
      blo[j][h2] = vl;
    }
  // z term: sum_c q1_c z_c (quad reduction), broadcast to the C-fragment rows.
  int zq = 0;
#pragma unroll
  for (int i = 0; i < HD / 64; ++i) {
    const uint4 zv = *reinterpret_cast<const uint4*>(rec + HD + q * R + 16 * i);
    zq = __dp4a((int)zv.x, (int)q1r[i].x, zq);
    zq = __dp4a((int)zv.y, (int)q1r[i].y, zq);
    zq = __dp4a((int)zv.z, (int)q1r[i].z, zq);
    zq = __dp4a((int)zv.w, (int)q1r[i].w, zq);
  }
  zq += __shfl_xor_sync(0xffffffffu, zq, 1);
  zq += __shfl_xor_sync(0xffffffffu, zq, 2);
  const int z0 = __shfl_sync(0xffffffffu, zq, 8 * q), z1 = __shfl_sync(0xffffffffu, zq, 8 * q + 4);
  // A fragments: raw codes of tokens 16 mt + g (+8), the lane's channel region.
  const uint8_t* codes = rec + 2 * HD;
  constexpr int TB = HD * BK / 8;   // bytes per token
  constexpr int QB = TB / 4;        // bytes per lane region
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    int ch[4] = {0, 0, 0, 0}, cl[4] = {0, 0, 0, 0};
    uint32_t w0[QB / 4], w1[QB / 4];
    const uint8_t* t0 = codes + (16 * mt + g) * TB + q * QB;
    const uint8_t* t1 = t0 + 8 * TB;
#pragma unroll
    for (int i = 0; i < QB / 4; ++i) {
      w0[i] = reinterpret_cast<const uint32_t*>(t0)[i];
      w1[i] = reinterpret_cast<const uint32_t*>(t1)[i];
    }
#pragma unroll
    for (int j = 0; j < KS; ++j) {
      uint32_t af[4];
      if (BK == 4) {
        af[0] = w0[j] & 0x0F0F0F0Fu;
        af[1] = w1[j] & 0x0F0F0F0Fu;
        af[2] = (w0[j] >> 4) & 0x0F0F0F0Fu;
        af[3] = (w1[j] >> 4) & 0x0F0F0F0Fu;
      } else {
        const int sh = 4 * (j & 1);
        af[0] = (w0[j >> 1] >> sh) & 0x03030303u;
        af[1] = (w1[j >> 1] >> sh) & 0x03030303u;
        af[2] = (w0[j >> 1] >> (sh + 2)) & 0x03030303u;
        af[3] = (w1[j >> 1] >> (sh + 2)) & 0x03030303u;
      }
      const uint32_t bh[2] = {bhi[j][0], bhi[j][1]}, bl[2] = {blo[j][0], blo[j][1]};
      imma_u8s8(ch, af, bh);
      imma_u8u8(cl, af, bl);
    }
    s[mt][0] = 128 * ch[0] + cl[0] + z0;
    s[mt][1] = 128 * ch[1] + cl[1] + z1;
    s[mt][2] = 128 * ch[2] + cl[2] + z0;
    s[mt][3] = 128 * ch[3] + cl[3] + z1;
  }
}

template <int HD, int BV>
TA_DEV void pv_q2(const uint8_t* rec, uint8_t (*pbuf)[kBc], const int (&sum_p)[2], int (&acc)[HD / 16][4], int g,
                  int q) {
  const uint8_t* codes = rec + 2 * HD;
  constexpr int CB = kBc * BV / 8;  // bytes per channel
  uint32_t bf[2][2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    bf[j][0] = *reinterpret_cast<const uint32_t*>(&pbuf[g][32 * j + 4 * q]);
    bf[j][1] = *reinterpret_cast<const uint32_t*>(&pbuf[g][32 * j + 16 + 4 * q]);
  }
#pragma unroll
  for (int mt = 0; mt < HD / 16; ++mt) {
    const int c0 = 16 * mt + g, c1 = c0 + 8;
    int c[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      uint32_t af[4];
      if (BV == 4) {
        const uint32_t u0 = reinterpret_cast<const uint32_t*>(codes + c0 * CB)[4 * j + q];
        const uint32_t u1 = reinterpret_cast<const uint32_t*>(codes + c1 * CB)[4 * j + q];
        af[0] = u0 & 0x0F0F0F0Fu;
        af[1] = u1 & 0x0F0F0F0Fu;
        af[2] = (u0 >> 4) & 0x0F0F0F0Fu;
        af[3] = (u1 >> 4) & 0x0F0F0F0Fu;
      } else {
        const uint32_t u0 = reinterpret_cast<const uint32_t*>(codes + c0 * CB)[q];
        const uint32_t u1 = reinterpret_cast<const uint32_t*>(codes + c1 * CB)[q];
        const int sh = 4 * j;
        af[0] = (u0 >> sh) & 0x03030303u;
        af[1] = (u1 >> sh) & 0x03030303u;
        af[2] = (u0 >> (sh + 2)) & 0x03030303u;
        af[3] = (u1 >> (sh + 2)) & 0x03030303u;
      }
      const uint32_t b[2] = {bf[j][0], bf[j][1]};
      imma_u8u8(c, af, b);
    }
    const int s0 = rec[c0], s1 = rec[c1];
    const int z0 = (int)(int8_t)rec[HD + c0], z1 = (int)(int8_t)rec[HD + c1];
    acc[mt][0] = s0 * c[0] + z0 * sum_p[0];
    acc[mt][1] = s0 * c[1] + z0 * sum_p[1];
    acc[mt][2] = s1 * c[2] + z1 * sum_p[0];
    acc[mt][3] = s1 * c[3] + z1 * sum_p[1];
  }
}

template <int HD>
__global__ void __launch_bounds__(32 * kWarpsPerCta) decode_kernel(const __grid_constant__ DecodeArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  DecodeWarpSmem<HD>& sm = reinterpret_cast<DecodeWarpSmem<HD>*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127))[warp];
  const int task = blockIdx.x * kWarpsPerCta + warp;
  if (task >= a.B * a.Hkv * a.n_splits) return;
  const int split = task % a.n_splits, bh = task / a.n_splits, b = bh / a.Hkv, kvh = bh % a.Hkv;
  const int G = a.G;
  const int nb = a.counters[2 * b], nbuf = a.counters[2 * b + 1];
  const int jb = min(a.blk_begin, nb), je = a.blk_end < 0 ? nb : min(a.blk_end, nb);
  const int nblk = max(0, je - jb), per = (nblk + a.n_splits - 1) / a.n_splits;
  const int j0 = min(jb + split * per, je), j1 = min(j0 + per, je);
  const bool use_buf = a.with_buffer && split == a.n_splits - 1 && nbuf > 0;
  const int bitsK = a.bits[kvh * 2], bitsV = a.bits[kvh * 2 + 1];
  const size_t slotK = ((size_t)b * a.Hkv + kvh) * 2, slotV = slotK + 1;
  constexpr int REC = rec_bytes(HD);
  const uint32_t bytesK = 2 * HD + kBc * HD * bitsK / 8, bytesV = 2 * HD + kBc * HD * bitsV / 8;
  const float lut_lane = sas_lut_lane(a.sas, lane);
  const int tap_row = a.has_tap && split == 0 && a.tap.batch == b && a.tap.head / G == kvh ? a.tap.head % G : -1;

  if (lane == 0) {
    mbar_init(&sm.bar[0], 1);
    mbar_init(&sm.bar[1], 1);
    fence_barrier_init();
  }
  __syncwarp();
  auto issue = [&](int j, int stg) {
    if (lane == 0) {
      mbar_expect_tx(&sm.bar[stg], bytesK + bytesV);
      bulk_load(sm.rec[stg][0], a.block_rec + (slotK * a.max_blocks + j) * REC, bytesK, &sm.bar[stg]);
      bulk_load(sm.rec[stg][1], a.block_rec + (slotV * a.max_blocks + j) * REC, bytesV, &sm.bar[stg]);
    }
  };
  if (j0 < j1) issue(j0, 0);
  if (j0 + 1 < j1) issue(j0 + 1, 1);

  // q stage-1 quantisation per (b, head) vector (Alg. 2).
  float s_q_row = 0.f;
  {
    const int R = HD / 4;
    float qa = 0.f;
    float xv[HD / 4];
    const __half* qp = a.q + ((size_t)b * a.Hq + kvh * G + g) * HD + q * R;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      xv[i] = g < G ? __half2float(qp[i]) : 0.f;
      qa = fmaxf(qa, fabsf(xv[i]));
    }
    qa = fmaxf(qa, __shfl_xor_sync(0xffffffffu, qa, 1));
    qa = fmaxf(qa, __shfl_xor_sync(0xffffffffu, qa, 2));
    const float inv = qa > 0.f ? __fdiv_rn(kDiv, qa) : 0.f;
    s_q_row = __fdiv_rn(qa, kDiv);
#pragma unroll
    for (int i = 0; i < R; ++i) sm.q1[g][q * R + i] = (int8_t)rint_prod(xv[i], inv);
    if (g == tap_row) {
      for (int i = 0; i < R; ++i) a.tap.q1[q * R + i] = sm.q1[g][q * R + i];
      if (q == 0) a.tap.s_q[0] = s_q_row;
    }
  }
  __syncwarp();
  uint4 q1r[HD / 64];  // the lane's channel region of row g
#pragma unroll
  for (int i = 0; i < HD / 64; ++i) q1r[i] = *reinterpret_cast<const uint4*>(&sm.q1[g][q * (HD / 4) + 16 * i]);
  const float sq2[2] = {__shfl_sync(0xffffffffu, s_q_row, 8 * q), __shfl_sync(0xffffffffu, s_q_row, 8 * q + 4)};

  RowState<HD> st;
  st.m[0] = st.m[1] = -INFINITY;
  st.l[0] = st.l[1] = 0.f;
#pragma unroll
  for (int mt = 0; mt < HD / 16; ++mt)
#pragma unroll
    for (int i = 0; i < 4; ++i) st.o[mt][i] = 0.f;

  for (int j = j0; j < j1; ++j) {
    const int stg = (j - j0) & 1;
    mbar_wait(&sm.bar[stg], ((j - j0) >> 1) & 1);
    const uint8_t* recK = sm.rec[stg][0];
    const uint8_t* recV = sm.rec[stg][1];
    int s[4][4];
    if (bitsK == 4) qk_q2<HD, 4>(recK, q1r, s, g, q);
    else qk_q2<HD, 2>(recK, q1r, s, g, q);
    const float sK = a.s_parent[slotK * a.max_blocks + j], sV = a.s_parent[slotV * a.max_blocks + j];
    const float cqk[2] = {__fmul_rn(__fmul_rn(sq2[0], sK), a.scale), __fmul_rn(__fmul_rn(sq2[1], sK), a.scale)};
    const bool tap = tap_row >= 0 && a.tap.j_block == j;
    if (tap) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int mt = i >> 1, hi = i & 1;
        const int e = tap_row - 2 * q;
        if (e == 0 || e == 1) a.tap.s_int[16 * mt + g + 8 * hi] = s[mt][2 * hi + e];
      }
    }
    float alpha[2], s_p[2];
    int sum_p[2];
    softmax_tile<HD>(a, st, s, kBc, cqk, sm.p, lut_lane, alpha, s_p, sum_p, tap, tap_row, g, q);
    int acc[HD / 16][4];
    if (bitsV == 4) pv_q2<HD, 4>(recV, sm.p, sum_p, acc, g, q);
    else pv_q2<HD, 2>(recV, sm.p, sum_p, acc, g, q);
    if (tap) {
      const int e = tap_row - 2 * q;
      if (e == 0 || e == 1)
#pragma unroll
        for (int mt = 0; mt < HD / 16; ++mt) {
          a.tap.pv_int[16 * mt + g] = acc[mt][e];
          a.tap.pv_int[16 * mt + g + 8] = acc[mt][2 + e];
        }
    }
    const float cpv[2] = {__fmul_rn(s_p[0], sV), __fmul_rn(s_p[1], sV)};
    pv_update<HD>(st, acc, alpha, cpv);
    __syncwarp();
    if (j + 2 < j1) issue(j + 2, stg);
  }

  if (use_buf) {
    // Buffer block (INT8, universal scale, n_buf valid keys), last.
    const int8_t* kb = a.buf + slotK * (size_t)(kBc * HD);
    const int8_t* vb = a.buf + slotV * (size_t)(kBc * HD);
    const float sK = __fdiv_rn(a.a_univ[slotK], kDiv), sV = __fdiv_rn(a.a_univ[slotV], kDiv);
    int s[4][4];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      int c[4] = {0, 0, 0, 0};
#pragma unroll
      for (int j = 0; j < HD / 32; ++j) {
        const int t0 = 16 * mt + g, t1 = t0 + 8;
        uint32_t af[4];
        af[0] = *reinterpret_cast<const uint32_t*>(kb + t0 * HD + 32 * j + 4 * q);
        af[1] = *reinterpret_cast<const uint32_t*>(kb + t1 * HD + 32 * j + 4 * q);
        af[2] = *reinterpret_cast<const uint32_t*>(kb + t0 * HD + 32 * j + 16 + 4 * q);
        af[3] = *reinterpret_cast<const uint32_t*>(kb + t1 * HD + 32 * j + 16 + 4 * q);
        const uint32_t bq[2] = {*reinterpret_cast<const uint32_t*>(&sm.q1[g][32 * j + 4 * q]),
                                *reinterpret_cast<const uint32_t*>(&sm.q1[g][32 * j + 16 + 4 * q])};
        imma_s8s8(c, af, bq);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) s[mt][i] = c[i];
    }
    const float cqk[2] = {__fmul_rn(__fmul_rn(sq2[0], sK), a.scale), __fmul_rn(__fmul_rn(sq2[1], sK), a.scale)};
    const bool tap = tap_row >= 0 && a.tap.j_block == -1;
    if (tap) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int mt = i >> 1, hi = i & 1, e = tap_row - 2 * q, tok = 16 * mt + g + 8 * hi;
        if (e == 0 || e == 1) a.tap.s_int[tok] = tok < nbuf ? s[mt][2 * hi + e] : 0;
      }
    }
    float alpha[2], s_p[2];
    int sum_p[2];
    softmax_tile<HD>(a, st, s, nbuf, cqk, sm.p, lut_lane, alpha, s_p, sum_p, tap, tap_row, g, q);
    int acc[HD / 16][4];
    uint32_t bf[2][2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      bf[j][0] = *reinterpret_cast<const uint32_t*>(&sm.p[g][32 * j + 4 * q]);
      bf[j][1] = *reinterpret_cast<const uint32_t*>(&sm.p[g][32 * j + 16 + 4 * q]);
    }
#pragma unroll
    for (int mt = 0; mt < HD / 16; ++mt) {
      const int c0 = 16 * mt + g, c1 = c0 + 8;
      int c[4] = {0, 0, 0, 0};
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        uint32_t af[4];
        af[0] = *reinterpret_cast<const uint32_t*>(vb + c0 * kBc + 32 * j + 4 * q);
        af[1] = *reinterpret_cast<const uint32_t*>(vb + c1 * kBc + 32 * j + 4 * q);
        af[2] = *reinterpret_cast<const uint32_t*>(vb + c0 * kBc + 32 * j + 16 + 4 * q);
        af[3] = *reinterpret_cast<const uint32_t*>(vb + c1 * kBc + 32 * j + 16 + 4 * q);
        const uint32_t b2[2] = {bf[j][0], bf[j][1]};
        imma_s8u8(c, af, b2);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[mt][i] = c[i];
    }
    if (tap) {
      const int e = tap_row - 2 * q;
      if (e == 0 || e == 1)
#pragma unroll
        for (int mt = 0; mt < HD / 16; ++mt) {
          a.tap.pv_int[16 * mt + g] = acc[mt][e];
          a.tap.pv_int[16 * mt + g + 8] = acc[mt][2 + e];
        }
    }
    const float cpv[2] = {__fmul_rn(s_p[0], sV), __fmul_rn(s_p[1], sV)};
    pv_update<HD>(st, acc, alpha, cpv);
  }

  // O = diag(l)^-1 O, L = m + log l; empty -> O = 0, L = -inf.
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int row = 2 * q + e;
    if (row >= G) continue;
    const bool empty = st.l[e] == 0.f;
    const float inv_l = empty ? 0.f : 1.f / st.l[e];
    const size_t orow = (size_t)b * a.Hq + kvh * G + row;
    const size_t base = ((size_t)split * a.B * a.Hq + orow) * HD;
#pragma unroll
    for (int mt = 0; mt < HD / 16; ++mt) {
      const float v0 = st.o[mt][e] * inv_l, v1 = st.o[mt][2 + e] * inv_l;
      if (a.o_parts) {
        a.o_parts[base + 16 * mt + g] = v0;
        a.o_parts[base + 16 * mt + g + 8] = v1;
      }
      if (a.o16) {
        a.o16[orow * HD + 16 * mt + g] = __float2half_rn(v0);
        a.o16[orow * HD + 16 * mt + g + 8] = __float2half_rn(v1);
      }
    }
    if (g == 0) a.lse_parts[(size_t)split * a.B * a.Hq + orow] = empty ? -INFINITY : st.m[e] + logf(st.l[e]);
  }
}

// Log-sum-exp combine over parts in ascending order (R-23).  One thread per
// (row, channel).
__global__ void combine_kernel(int n_parts, int rows, int d, const float* __restrict__ o_parts,
                               const float* __restrict__ lse_parts, __half* __restrict__ o16,
                               float* __restrict__ o32, float* __restrict__ lse) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * d) return;
  const int r = idx / d, c = idx % d;
  float lmax = -INFINITY;
  for (int s = 0; s < n_parts; ++s) lmax = fmaxf(lmax, lse_parts[(size_t)s * rows + r]);
  float out = 0.f, L = -INFINITY;
  if (lmax != -INFINITY) {
    float wsum = 0.f;
    for (int s = 0; s < n_parts; ++s) wsum += expf(lse_parts[(size_t)s * rows + r] - lmax);
    const float inv = 1.f / wsum;
    for (int s = 0; s < n_parts; ++s)
      out += expf(lse_parts[(size_t)s * rows + r] - lmax) * inv * o_parts[((size_t)s * rows + r) * d + c];
    L = lmax + logf(wsum);
  }
  if (o16) o16[(size_t)r * d + c] = __float2half_rn(out);
  if (o32) o32[(size_t)r * d + c] = out;
  if (c == 0) lse[r] = L;
}

}  // namespace ta

namespace ta_host {
using namespace ta;

size_t decode_workspace(int B, int Hq, int HD, int S) {
  if (S <= 1) return 0;
  return (size_t)S * B * Hq * (HD + 1) * sizeof(float);
}

cudaError_t launch_decode(const turbo_params_t* p, const turbo_kv_cache_t* c, int Hq, const __half* q, int blk_begin,
                          int blk_end, int with_buffer, int S, void* ws, __half* o, float* o_part, float* lse,
                          cudaStream_t st) {
  const int B = c->batch, H = c->n_kv_heads, HD = c->head_dim;
  DecodeArgs a;
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
  a.scale = p->softmax_scale;
  fill_sas_const(&a.sas, p->sas_nr);
  a.has_tap = p->debug_tap != nullptr;
  if (a.has_tap) a.tap = *reinterpret_cast<const turbo_debug_tap_t*>(p->debug_tap);
  else memset(&a.tap, 0, sizeof(a.tap));
  if (S == 1) {
    a.o_parts = o_part;
    a.lse_parts = lse;
    a.o16 = o;
  } else {
    a.o_parts = reinterpret_cast<float*>(ws);
    a.lse_parts = a.o_parts + (size_t)S * B * Hq * HD;
    a.o16 = nullptr;
  }
  const int tasks = B * H * S;
  const dim3 grid((tasks + kWarpsPerCta - 1) / kWarpsPerCta);
  if (HD == 128) {
    const size_t smem = sizeof(DecodeWarpSmem<128>) * kWarpsPerCta + 128;
    cudaFuncSetAttribute(decode_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    decode_kernel<128><<<grid, 32 * kWarpsPerCta, smem, st>>>(a);
  } else {
    const size_t smem = sizeof(DecodeWarpSmem<64>) * kWarpsPerCta + 128;
    cudaFuncSetAttribute(decode_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    decode_kernel<64><<<grid, 32 * kWarpsPerCta, smem, st>>>(a);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || S == 1) return e;
  const int rows = B * Hq;
  combine_kernel<<<(rows * HD + 255) / 256, 256, 0, st>>>(S, rows, HD, a.o_parts, a.lse_parts, o, o_part, lse);
  return cudaGetLastError();
}

cudaError_t launch_combine(int n_parts, int rows, int d, const float* o_parts, const float* lse_parts, __half* o,
                           float* o32, float* lse, cudaStream_t st) {
  combine_kernel<<<(rows * d + 255) / 256, 256, 0, st>>>(n_parts, rows, d, o_parts, lse_parts, o, o32, lse);
  return cudaGetLastError();
}
}  // namespace ta_host
