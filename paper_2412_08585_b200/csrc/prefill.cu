// prefill.cu -- Algorithm 1 (TurboAttention prefill) on sm_100a.
//
// One CTA = one (batch, pair of GQA query heads sharing a KV head, 128-row
// query tile); each tile holds two B_r = 64 quantisation blocks (or one
// B_r = 128 block).  One CTA per SM (all 512 TMEM columns).  Warp roles:
//   warp 0      TMA producer: K_j [64 x d] INT8 and V_j^T [d x 64] FP16-code
//               tiles into a 3-stage smem ring shared by both query tiles
//               (cp.async.bulk.tensor, 128B/64B swizzle).
//   warps 1, 2  one single-thread tcgen05.mma issuer per query tile (warp 1
//               also owns TMEM): S_j = Q^q1 K_j^q1^T (kind::i8 -> int32 TMEM,
//               double-buffered) and PV_j = Q(P~_j) V_j^q1 (kind::f16 on the
//               exact integer codes -> fp32 TMEM, exact).
//   warps 4-11  one softmax warpgroup per query tile, thread = query row =
//               TMEM lane: Q stage-1 quantisation, x and the row max (pass 1),
//               SAS (LUT x POLY) + row sum + P max (pass 2), P tile scale and
//               codes -> smem, the A operand of the PV MMA (pass 3), and
//               O += (s_P s_V / A) PV_int in FP32 registers one tile behind;
//               the epilogue writes O through smem (row-contiguous stores).
#include <algorithm>
#include <climits>
#include <cstring>

#include "common.cuh"

#ifdef TURBO_PROFILE
__device__ unsigned long long g_prof[32];
// per-thread register accumulators, flushed once per CTA (global atomics per
// event would serialise the SMs and distort the timeline)
#define PROF_T(var) const long long var = clock64()
#define PROF_ADD(slot, a, b) prof_acc[slot] += (uint32_t)((b) - (a))
#else
#define PROF_T(var)
#define PROF_ADD(slot, a, b)
#endif

namespace ta {

constexpr int kStages = 3;
constexpr int kTileM = 128;
#ifndef TA_PREFILL_SPLIT
#define TA_PREFILL_SPLIT 1  // softmax warps per 32-row quadrant (2 = column halves; measured slower)
#endif

// NS query tiles ("slots") per CTA share every K/V tile: NS = 2 pairs two
// query heads of the same KV head (GQA) at the same rows, each with its own
// softmax warpgroup, S/PV TMEM columns and P buffers.  For odd G (MHA) the two
// slots are adjacent query tiles 2i, 2i+1 of one head (TP): they share all K/V
// tiles but the last <= 2, which the lower tile sees fully masked -- 474 vs 345
// TOPS for one tile per CTA (8 x 4096, 32 heads, d = 128).
template <int HD, int NS, int SP>
struct PrefillSmem {
  int8_t q1[NS][kTileM * HD];       // Q^q1, K-major, swizzled rows of HD bytes
  int8_t k[kStages][kBc * HD];      // K_j^q1 [64][HD]
  __half v[kStages][HD * kBc];      // V_j^q1 codes as fp16, transposed [HD][64] (128-B rows, SW128)
  __half p[NS][2][kTileM * kBc];    // Q(P~) codes as fp16 [128][64] (128-B rows, SW128)
  uint64_t kv_full[kStages], kv_empty[kStages];
  uint64_t s_full[NS][2], s_free[NS][2], p_full[NS][2], pv_full[NS], pv_free[NS], q_ready;
  uint64_t pmax_bar[NS][2];  // per P-scale group: arrivals of its warps' partial max
  uint32_t tmem_base;
  float red_a[NS][4][SP];
  float red_p[NS][2][4 * SP];
  float xmax[NS][2][SP][kTileM];  // per-half row max exchange (SP = 2)
  float lsum[NS][SP][kTileM];     // per-half row sums (SP = 2)
};

struct PrefillArgs {
  const __half* q;
  __half* o;
  float* lse;
  const float* k1s;
  const float* v1s;
  int B, N, Hq, Hkv, causal, block_q, alpha_mode, n_qtiles, unit_group;
  int Nk, q0;  // keys per sequence; absolute position of query row 0 (chunked prefill: Nk - N)
  float scale;
  SasConst sas;
  int has_tap;
  turbo_debug_tap_t tap;
};

template <int HD>
TA_DEV uint32_t q1_swz(int r, int chunk) {
  // 128B swizzle for 128-B rows, 64B swizzle for 64-B rows (matches the TMA
  // swizzle of the K tile and the UMMA descriptor layout type).
  if (HD == 128) return r * 128 + ((chunk ^ (r & 7)) << 4);
  return r * 64 + ((chunk ^ ((r >> 1) & 3)) << 4);
}
TA_DEV uint32_t p_swz(int r, int chunk) { return r * 128 + ((chunk ^ (r & 7)) << 4); }  // SW128, 16-B chunk of 8 halves

// Register split between the control warpgroup and the softmax warpgroups.
// setmaxnreg.inc can only take registers released by setmaxnreg.dec of the
// same CTA, so  128 * dec + 128 * NS * SP * inc <= threads * launch_regs.
template <int NS, int SP>
TA_DEV void reg_dealloc() {
  if (NS * SP == 2) asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");  // 384 thr x 168
  if (NS * SP == 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 24;\n" ::: "memory");  // 640 thr x 96
}
template <int NS, int SP>
TA_DEV void reg_alloc() {
  if (NS * SP == 2) asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
  if (NS * SP == 4) asm volatile("setmaxnreg.inc.sync.aligned.u32 112;\n" ::: "memory");
}

template <int HD, int NS, int SP, bool TAP, bool TP>
__global__ void __launch_bounds__(128 * (1 + NS * SP), 1)
    prefill_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                   const __grid_constant__ PrefillArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
#ifdef TURBO_PROFILE
  const long long t_cta0 = clock64();
  uint32_t prof_acc[17] = {0};
#endif
  using Smem = PrefillSmem<HD, NS, SP>;
  // 1024-B aligned (128B-swizzle atoms); pointer arithmetic keeps the shared address space.
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t kTmemCols = NS == 2 ? 512 : 256;  // per slot: S0 [0,64) S1 [64,128) PV [128,128+d)

  // Work item: (query tile, batch, kv head, head group of NS).  Units are
  // taken in groups of UG (about 4 x 148 CTAs' worth), heaviest (last) query
  // tiles first inside a group for causal load balance; the group keeps the
  // K/V streams resident in L2 (DRAM reads = the compulsory bytes, down from
  // 2.9x with one global heavy-first order; same speed).
  // tile_pair (odd G): the two slots hold adjacent query tiles of the same head instead of
  // two heads of a GQA group; n_qtiles then counts tile pairs.
  constexpr bool tp = NS == 2 && TP;
  const int G = args.Hq / args.Hkv, GS = tp ? G : G / NS;
  const int units = args.B * args.Hkv * GS;
  const int UG = args.unit_group;
  const int grp_i = (int)blockIdx.x / (UG * args.n_qtiles), rem = (int)blockIdx.x % (UG * args.n_qtiles);
  const int UGg = min(UG, units - grp_i * UG);
  const int it = args.n_qtiles - 1 - rem / UGg;
  const int u = grp_i * UG + rem % UGg, b = u / (args.Hkv * GS), kvh = (u / GS) % args.Hkv, hg = u % GS;
  const int h0 = kvh * G + hg * (tp ? 1 : NS);
  const int N = args.N, Tc = (args.Nk + kBc - 1) / kBc;  // N query rows, Tc key tiles
  // query tile of slot s and the key tiles it visits (0 for a tile past the end)
  auto tile_of = [&](int s) { return tp ? 2 * it + s : it; };
  auto nkv_of = [&](int s) {
    const int ti = tile_of(s);
    if (ti * kTileM >= N) return 0;
    const int last_row = min(ti * kTileM + kTileM - 1, N - 1);
    return args.causal ? min(Tc, (args.q0 + last_row) / kBc + 1) : Tc;
  };
  const int nkv = NS == 2 ? max(nkv_of(0), nkv_of(1)) : nkv_of(0);  // tiles the CTA streams
  const size_t bkv = (size_t)b * args.Hkv + kvh;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.kv_full[s], 1);
      mbar_init(&sm.kv_empty[s], NS);  // one commit per MMA issuer
    }
    for (int t = 0; t < NS; ++t) {
      for (int s = 0; s < 2; ++s) {
        mbar_init(&sm.s_full[t][s], 1);
        mbar_init(&sm.s_free[t][s], 128 * SP);
        mbar_init(&sm.p_full[t][s], 128 * SP);
      }
      mbar_init(&sm.pv_full[t], 1);
      mbar_init(&sm.pv_free[t], 128 * SP);
      for (int g2 = 0; g2 < 2; ++g2) mbar_init(&sm.pmax_bar[t][g2], (args.block_q / 32) * SP);
    }
    mbar_init(&sm.q_ready, 128 * NS * SP);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&sm.tmem_base, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp < 4) {
    reg_dealloc<NS, SP>();
    if (warp == 0) {
      // ---------------------------------------------------------- TMA producer
      if (elect_one()) {
        tma_prefetch_desc(&tm_k);
        tma_prefetch_desc(&tm_v);
        for (int j = 0; j < nkv; ++j) {
          const int st = j % kStages, n = j / kStages;
          PROF_T(w0);
          if (n > 0) mbar_wait(&sm.kv_empty[st], (n - 1) & 1);
          PROF_T(w1);
          PROF_ADD(16, w0, w1);
          mbar_expect_tx(&sm.kv_full[st], 3 * kBc * HD);  // K int8 + V fp16
          tma_load_3d(sm.k[st], &tm_k, &sm.kv_full[st], 0, j * kBc, (int)bkv);
          tma_load_3d(sm.v[st], &tm_v, &sm.kv_full[st], 0, 0, (int)(bkv * Tc + j));
        }
      }
    } else if (warp == 1 || (NS == 2 && warp == 2)) {
      // ---------------------------------------------------------- MMA issuers
      // One issuing warp per query tile (warp 1: slot 0, warp 2: slot 1), so a slot
      // whose softmax runs ahead is not held behind the other slot's P tile.
      const int t = warp - 1;
      constexpr uint32_t kLayQK = HD == 128 ? kSw128 : kSw64;
      constexpr uint32_t idesc_qk = idesc_i8(kTileM, kBc, true, true);
      // P V runs as kind::f16: codes are small integers (exact in fp16) and every
      // partial sum is an integer < 2^24, so the fp32 accumulator holds PV_int exactly.
      constexpr uint32_t idesc_pv = idesc_f16(kTileM, HD);
      mbar_wait(&sm.q_ready, 0);
      tc_fence_after();
      for (int j = 0; j <= nkv; ++j) {
        if (j < nkv) {
          const int st = j % kStages, sb = j & 1;
          PROF_T(m0);
          mbar_wait(&sm.kv_full[st], (j / kStages) & 1);
          PROF_T(m1);
          PROF_ADD(10, m0, m1);
          const uint32_t ka = smem_u32(sm.k[st]);
          {
            PROF_T(m2);
            if (j >= 2) mbar_wait(&sm.s_free[t][sb], ((j >> 1) - 1) & 1);
            PROF_T(m3);
            PROF_ADD(11, m2, m3);
            tc_fence_after();
            if (elect_one()) {
              const uint32_t q1a = smem_u32(sm.q1[t]);
#pragma unroll
              for (int ks = 0; ks < HD / 32; ++ks)
                mma_i8_ss(tmem + t * 256 + sb * kBc, smem_desc(q1a + ks * 32, 8 * HD, kLayQK),
                          smem_desc(ka + ks * 32, 8 * HD, kLayQK), idesc_qk, ks > 0);
              mma_commit(&sm.s_full[t][sb]);
            }
            __syncwarp();
          }
        }
        if (j >= 1) {
          const int jj = j - 1, pb = jj & 1, st = jj % kStages;
          const uint32_t va = smem_u32(sm.v[st]);
          {
            PROF_T(m4);
            mbar_wait(&sm.p_full[t][pb], (jj >> 1) & 1);
            PROF_T(m5);
            if (jj >= 1) mbar_wait(&sm.pv_free[t], (jj - 1) & 1);
            PROF_T(m6);
            PROF_ADD(12, m4, m5);
            PROF_ADD(13, m5, m6);
            tc_fence_after();
            if (elect_one()) {
              const uint32_t pa = smem_u32(sm.p[t][pb]);
#pragma unroll
              for (int ks = 0; ks < kBc / 16; ++ks)
                mma_f16_ss(tmem + t * 256 + 2 * kBc, smem_desc(pa + ks * 32, 1024, kSw128),
                           smem_desc(va + ks * 32, 1024, kSw128), idesc_pv, ks > 0);
              mma_commit(&sm.pv_full[t]);
              mma_commit(&sm.kv_empty[st]);
            }
            __syncwarp();
          }
        }
      }
    }
  } else {
    reg_alloc<NS, SP>();
    PROF_T(pro0);
    // ------------------------------------------------------------ softmax / correction
    // Thread = (slot, column half hc, row r = TMEM lane).  With SP = 2 two warps
    // share each 32-row quadrant: hc owns S columns [hc SW, (hc+1) SW) and O
    // columns [hc OW, (hc+1) OW); row max is exchanged per tile, partial row sums
    // are added at the end (l is linear in the halves).
    constexpr int SW = kBc / SP, OW = HD / SP, CW = SP == 2 ? 16 : 32;
    const int widx = warp - 4, slot = widx / (4 * SP), hc = (widx >> 2) % SP, h = tp ? h0 : h0 + slot;
    // tile_pair: both slots walk the CTA's nkv key tiles; the lower tile's last ones (<= 2)
    // are fully masked for it (kmax) and cost one inactive softmax pass each.
    const int its = tile_of(slot), nkv_s = nkv;
    const int qd = warp & 3, r = qd * 32 + lane, row = its * kTileM + r;
    const bool row_ok = row < N;
    const int half = args.block_q == 64 ? (r >> 6) : 0;
    const int grp = half;  // P-scale group (B_r rows)
    const uint32_t tbase = tmem + ((uint32_t)(qd * 32) << 16) + slot * 256;
    const float lut_lane = sas_lut_lane(args.sas, lane);
    const float nr_abs = args.sas.nr_abs;
    const bool tap_cta = TAP && args.tap.batch == b && args.tap.head == h &&
                         (args.tap.i_block >> 1) == its;
    const bool tap_row = tap_cta && (args.tap.i_block & 1) == (r >> 6);
    float* red_p = &sm.red_p[slot][0][0];
    const uint32_t bar_slot = 1 + slot;                // 128*SP threads of the slot
    const uint32_t bar_pair = 3 + slot * 4 + qd;       // the SP warps of one quadrant

    // Q stage-1 quantisation (Alg. 1; per B_r x d block): this thread
    // quantises the channels [hc OW, (hc+1) OW) of its row.
    float s_q;
    {
      uint4 qraw[OW / 8];
      float qa = 0.f;
      const __half* qrow = args.q + (((size_t)b * N + row) * args.Hq + h) * HD + hc * OW;
#pragma unroll
      for (int c = 0; c < OW / 8; ++c) {
        qraw[c] = row_ok ? reinterpret_cast<const uint4*>(qrow)[c] : make_uint4(0, 0, 0, 0);
        const __half2* hp = reinterpret_cast<const __half2*>(&qraw[c]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 f = __half22float2(hp[e]);
          qa = fmaxf(qa, fmaxf(fabsf(f.x), fabsf(f.y)));
        }
      }
      qa = warp_max(qa);
      if (lane == 0) sm.red_a[slot][qd][hc] = qa;
      named_bar_sync(bar_slot, 128 * SP);
      float a_q = 0.f;
#pragma unroll
      for (int x = 0; x < SP; ++x)
        a_q = args.block_q == 64 ? fmaxf(a_q, fmaxf(sm.red_a[slot][2 * half][x], sm.red_a[slot][2 * half + 1][x]))
                                 : fmaxf(a_q, fmaxf(fmaxf(sm.red_a[slot][0][x], sm.red_a[slot][1][x]),
                                                    fmaxf(sm.red_a[slot][2][x], sm.red_a[slot][3][x])));
      const float inv_q = a_q > 0.f ? div_119_by(a_q) : 0.f;
      s_q = div_by_119(a_q);
#pragma unroll
      for (int c = 0; c < OW / 16; ++c) {
        uint32_t w[4];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const __half2* hp = reinterpret_cast<const __half2*>(&qraw[2 * c + hh]);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            float2 f0 = __half22float2(hp[2 * e]), f1 = __half22float2(hp[2 * e + 1]);
            w[hh * 2 + e] = pack4_lo(rint_prod_bits(f0.x, inv_q), rint_prod_bits(f0.y, inv_q),
                                     rint_prod_bits(f1.x, inv_q), rint_prod_bits(f1.y, inv_q));
          }
        }
        const int chunk = hc * (OW / 16) + c;
        *reinterpret_cast<uint4*>(sm.q1[slot] + q1_swz<HD>(r, chunk)) = make_uint4(w[0], w[1], w[2], w[3]);
        if (tap_row)
          *reinterpret_cast<uint4*>(args.tap.q1 + (r & 63) * HD + chunk * 16) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      if (tap_row && (r & 63) == 0 && hc == 0) args.tap.s_q[0] = s_q;
    }
    fence_proxy_async();
    mbar_arrive(&sm.q_ready);
    PROF_T(pro1);
    PROF_ADD(7, pro0, pro1);

    // Output accumulator in scaled form O_true = A * Ohat (A = product of the
    // alphas since the last renormalisation), so a tile costs one FFMA per
    // element: Ohat += (s_P s_V / A) PV.  Rounding order of O is free (R-16).
    float O[OW];
#pragma unroll
    for (int c = 0; c < OW; ++c) O[c] = 0.f;
    float m = -INFINITY, l = 0.f, A = 1.f;
    float cpv_p = 0.f;
    bool tap_p = false;
    const int kmax = row_ok ? (args.causal ? args.q0 + row : args.Nk - 1) : -1;  // last visible key of this row

    for (int j = 0; j <= nkv_s; ++j) {
      float cpv = 0.f, alpha_j = 0.f, sp_j = 0.f;
      bool active_j = false;
      const bool tap_j = tap_row && args.tap.j_block == j;
      if (j < nkv_s) {
        const int sb = j & 1;
        const uint32_t tS = tbase + sb * kBc + hc * SW;  // this thread's S columns (reused for x, P~)
        PROF_T(p0);
        mbar_wait_spin(&sm.s_full[slot][sb], (j >> 1) & 1);
        tc_fence_after();
        PROF_T(p1);
        PROF_ADD(0, p0, p1);
        const int nvalid = max(0, min(kBc, kmax - j * kBc + 1));  // visible keys of the tile
        const int nv = max(0, min(SW, nvalid - hc * SW));            // ... in this half
        const bool active = nvalid > 0;
        const bool full = __all_sync(0xffffffffu, nv == SW);
        // x = S s_Q s_K / sqrt(d) (R-18); masked keys -> -inf.
        const float cqk = __fmul_rn(__fmul_rn(s_q, args.k1s[bkv * Tc + j]), args.scale);
        float mt = -INFINITY;
        // passes 1 and 3 take the whole 64-column row in one TMEM round trip (two x32
        // loads, one wait): they hold few other values, unlike pass 2
        constexpr int CW1 = SP == 1 ? 64 : CW;
#pragma unroll 1
        for (int ch = 0; ch < SW / CW1; ++ch) {
          uint32_t v[CW1];
#pragma unroll
          for (int h2 = 0; h2 < CW1 / CW; ++h2) TA_TMEM_LD(CW, tS + ch * CW1 + h2 * CW, (v + h2 * CW));
          tmem_ld_wait();
          if (tap_j)
            for (int c = 0; c < CW1; ++c)
              args.tap.s_int[(r & 63) * kBc + hc * SW + ch * CW1 + c] = ch * CW1 + c < nv ? (int)v[c] : 0;
          const f32x2 cq2 = pk2(cqk, cqk);
          if (full) {
#pragma unroll
            for (int c = 0; c < CW1; c += 2) {
              const f32x2 x2 = mul2(pk2((float)(int)v[c], (float)(int)v[c + 1]), cq2);
              const float x0 = lo2(x2), x1 = hi2(x2);
              mt = fmaxf(mt, fmaxf(x0, x1));
              v[c] = __float_as_uint(x0);
              v[c + 1] = __float_as_uint(x1);
            }
          } else {
#pragma unroll
            for (int c = 0; c < CW1; c += 2) {
              const f32x2 x2 = mul2(pk2((float)(int)v[c], (float)(int)v[c + 1]), cq2);
              const float x0 = ch * CW1 + c < nv ? lo2(x2) : -INFINITY;
              const float x1 = ch * CW1 + c + 1 < nv ? hi2(x2) : -INFINITY;
              mt = fmaxf(mt, fmaxf(x0, x1));
              v[c] = __float_as_uint(x0);
              v[c + 1] = __float_as_uint(x1);
            }
          }
#pragma unroll
          for (int h2 = 0; h2 < CW1 / CW; ++h2) TA_TMEM_ST(CW, tS + ch * CW1 + h2 * CW, (v + h2 * CW));
        }
        if (SP == 2) {  // row max over both halves
          sm.xmax[slot][sb][hc][r] = mt;
          named_bar_sync(bar_pair, 64);
          mt = fmaxf(mt, sm.xmax[slot][sb][hc ^ 1][r]);
        }
        PROF_T(p2);
        PROF_ADD(1, p1, p2);
        // m_new, alpha = SAS(m_prev - m_new) (R-15)
        const float m_new = fmaxf(m, mt);
        float alpha = sas_eval(__fsub_rn(m_new, m), lut_lane, nr_abs);
        if (m == -INFINITY) alpha = 0.f;
        else if (args.alpha_mode == 1 && m_new == m) alpha = 1.f;
        const float m_use = active ? m_new : 0.f;  // inactive row: every x = -inf -> P~ = 0
        tmem_st_wait();
        // P~ = SAS(x - m_new), in place in TMEM; two elements per
        // FADD2 / FFMA2 / FMUL2, bit-identical to the scalar sas_eval.
        float pmax = 0.f;
        f32x2 rsum2 = pk2(0.f, 0.f);
        {
          const f32x2 m2 = pk2(m_use, m_use), mg2 = pk2(kMagic, kMagic);
          const f32x2 c3 = pk2(-0.1025f, -0.1025f), c2 = pk2(0.4626f, 0.4626f), c1 = pk2(-0.9922f, -0.9922f),
                      c0 = pk2(0.9996f, 0.9996f);
#pragma unroll 1
          for (int ch = 0; ch < SW / CW; ++ch) {
            uint32_t v[CW];
            TA_TMEM_LD(CW, tS + ch * CW, v);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < CW; c += 2) {
              const f32x2 d2 = sub2(m2, pk2(__uint_as_float(v[c]), __uint_as_float(v[c + 1])));
              const f32x2 t2 = add2_rd(d2, mg2);           // kMagic + floor(d)
              const f32x2 f2 = sub2(d2, sub2(t2, mg2));    // d - floor(d), exact
              const float l0 = lut_shfl(lut_lane, __float_as_uint(lo2(t2)));
              const float l1 = lut_shfl(lut_lane, __float_as_uint(hi2(t2)));
              const f32x2 p2 = fma2(fma2(fma2(c3, f2, c2), f2, c1), f2, c0);
              const f32x2 lp = mul2(pk2(l0, l1), p2);
              const float pt0 = lo2(d2) > nr_abs ? 0.f : lo2(lp);
              const float pt1 = hi2(d2) > nr_abs ? 0.f : hi2(lp);
              rsum2 = add2(rsum2, pk2(pt0, pt1));
              pmax = fmaxf(pmax, fmaxf(pt0, pt1));
              v[c] = __float_as_uint(pt0);
              v[c + 1] = __float_as_uint(pt1);
            }
            TA_TMEM_ST(CW, tS + ch * CW, v);
          }
        }
        const float rsum = lo2(rsum2) + hi2(rsum2);
        if (active) {
          l = alpha * l + rsum;  // l = SAS(m_prev - m_new) l + rowsum(P~), this half's share
          m = m_new;
        }
        PROF_T(p3);
        PROF_ADD(2, p2, p3);
        // P scale over the B_r x B_c tile: publish this warp's max
        // now, pick the group max up after the previous tile's O update.
        pmax = warp_max(pmax);
        if (lane == 0) {
          red_p[(sb * 4 + qd) * SP + hc] = pmax;
          mbar_arrive(&sm.pmax_bar[slot][grp]);
        }
        alpha_j = alpha;
        active_j = active;
      }
      // O += (s_P s_V / A) Q(P~) V^q1 for the previous tile
      if (j >= 1) {
        PROF_T(c0);
        mbar_wait_spin(&sm.pv_full[slot], (j - 1) & 1);
        tc_fence_after();
        PROF_T(c1);
        PROF_ADD(3, c0, c1);
#pragma unroll
        for (int cc = 0; cc < OW / 32; ++cc) {  // 32 columns per TMEM round trip
          uint32_t pv[32];
          TA_TMEM_LD32(tbase + 2 * kBc + hc * OW + cc * 32, pv);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const f32x2 o2 = fma2(pk2(cpv_p, cpv_p), pk2(__uint_as_float(pv[e]), __uint_as_float(pv[e + 1])),
                                  pk2(O[cc * 32 + e], O[cc * 32 + e + 1]));
            O[cc * 32 + e] = lo2(o2);
            O[cc * 32 + e + 1] = hi2(o2);
          }
          if (tap_p) {
            for (int e = 0; e < 32; ++e)
              args.tap.pv_int[(r & 63) * HD + hc * OW + cc * 32 + e] = (int)__uint_as_float(pv[e]);
          }
        }
        tc_fence_before();
        if (j < nkv_s) mbar_arrive(&sm.pv_free[slot]);
        PROF_T(c2);
        PROF_ADD(4, c1, c2);
      }
      if (j < nkv_s) {
        const int sb = j & 1;
        const uint32_t tS = tbase + sb * kBc + hc * SW;
        tmem_st_wait();
        PROF_T(q0);
        mbar_wait_spin(&sm.pmax_bar[slot][grp], j & 1);
        PROF_T(q1);
        PROF_ADD(5, q0, q1);
        float a_p = 0.f;
#pragma unroll
        for (int x = 0; x < SP; ++x)
          a_p = args.block_q == 64
                    ? fmaxf(a_p, fmaxf(red_p[(sb * 4 + 2 * half) * SP + x], red_p[(sb * 4 + 2 * half + 1) * SP + x]))
                    : fmaxf(a_p, fmaxf(fmaxf(red_p[(sb * 4) * SP + x], red_p[(sb * 4 + 1) * SP + x]),
                                       fmaxf(red_p[(sb * 4 + 2) * SP + x], red_p[(sb * 4 + 3) * SP + x])));
        const float inv_p = a_p > 0.f ? div_119_by(a_p) : 0.f;
        const float s_p = div_by_119(a_p);
        // Q(P~) codes in [0, 119] as fp16 -> smem (A operand of the PV MMA)
        uint8_t* prow = reinterpret_cast<uint8_t*>(sm.p[slot][sb]);
        constexpr float kMagicF16 = 12582912.0f + 25600.0f;  // 1.5*2^23 + 0x6400
        const __half2 c1024 = __half2(__float2half_rn(1024.f), __float2half_rn(1024.f));
        constexpr int CW3 = SP == 1 ? 64 : CW;
#pragma unroll 1
        for (int ch = 0; ch < SW / CW3; ++ch) {
          uint32_t v[CW3];
#pragma unroll
          for (int h2 = 0; h2 < CW3 / CW; ++h2) TA_TMEM_LD(CW, tS + ch * CW3 + h2 * CW, (v + h2 * CW));
          tmem_ld_wait();
#pragma unroll
          for (int hh = 0; hh < CW3 / 8; ++hh) {
            // y = 1.5*2^23 + 0x6400 + code: its low half-word is the fp16 of 1024 + code
            uint32_t y[8];
            const f32x2 inv2 = pk2(inv_p, inv_p), mf2 = pk2(kMagicF16, kMagicF16);
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              const f32x2 y2 = fma2(pk2(__uint_as_float(v[8 * hh + e]), __uint_as_float(v[8 * hh + e + 1])), inv2, mf2);
              y[e] = __float_as_uint(lo2(y2));
              y[e + 1] = __float_as_uint(hi2(y2));
            }
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const uint32_t hb = __byte_perm(y[2 * e], y[2 * e + 1], 0x5410);
              const __half2 hv = __hsub2(*reinterpret_cast<const __half2*>(&hb), c1024);  // exact
              w[e] = *reinterpret_cast<const uint32_t*>(&hv);
            }
            const int chunk = (hc * SW + ch * CW3) / 8 + hh;
            *reinterpret_cast<uint4*>(prow + p_swz(r, chunk)) = make_uint4(w[0], w[1], w[2], w[3]);
            if (tap_j)
              *reinterpret_cast<uint2*>(args.tap.p_codes + (r & 63) * kBc + chunk * 8) =
                  make_uint2(pack4_lo(y[0], y[1], y[2], y[3]), pack4_lo(y[4], y[5], y[6], y[7]));
          }
        }
        tc_fence_before();
        mbar_arrive(&sm.s_free[slot][sb]);
        if (tap_j && hc == 0) {
          args.tap.m_new[r & 63] = m;
          if ((r & 63) == 0) args.tap.s_p[0] = s_p;
        }
        fence_proxy_async();
        mbar_arrive(&sm.p_full[slot][sb]);
        sp_j = s_p;
        PROF_T(q2);
        PROF_ADD(6, q1, q2);
      }
      // Scaled-O bookkeeping, after PV(j-1) has landed in Ohat: O_true = A * Ohat,
      // tile j's alpha multiplies everything accumulated so far; fold A
      // into Ohat when it would underflow (alpha == 0 restarts the history).
      if (j < nkv_s && active_j) {
        const float An = A * alpha_j;
        if (!(An >= 1e-30f)) {
#pragma unroll
          for (int c = 0; c < OW; ++c) O[c] *= An;
          A = 1.f;
        } else {
          A = An;
        }
        cpv = __fdividef(__fmul_rn(sp_j, args.v1s[bkv * Tc + j]), A);  // tolerance set (R-16): ~2 ulp is fine
      }
      cpv_p = cpv;
      tap_p = tap_j;
    }
    PROF_T(epi0);
    if (SP == 2) {  // l = l_0 + l_1 (fixed order)
      sm.lsum[slot][hc][r] = l;
      named_bar_sync(bar_pair, 64);
      l = sm.lsum[slot][0][r] + sm.lsum[slot][1][r];
    }
    // Epilogue: O_i = diag(l)^-1 O, L_i = m + log l
    if (SP == 1) {
      // O rows go through shared memory (this warp's 32 rows in the now idle P buffers,
      // XOR-swizzled 16-byte chunks) so that the global stores are row-contiguous: one
      // instruction writes two whole 2d-byte rows instead of 32 scattered 16-byte pieces.
      constexpr int CH = HD / 8;  // 16-byte chunks per row
      uint8_t* stg = reinterpret_cast<uint8_t*>(sm.p[slot][qd >> 1]) + (qd & 1) * (32 * HD * 2);
      const float f = row_ok ? A / l : 0.f;
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        __half2 hv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) hv[e] = __floats2half2_rn(O[c * 8 + 2 * e] * f, O[c * 8 + 2 * e + 1] * f);
        *reinterpret_cast<uint4*>(stg + lane * (HD * 2) + ((c ^ (lane % CH)) << 4)) = *reinterpret_cast<uint4*>(hv);
      }
      __syncwarp();
      constexpr int RPI = 32 / CH;  // rows per store instruction
#pragma unroll
      for (int i = 0; i < 32 / RPI; ++i) {
        const int rr = RPI * i + lane / CH, c = lane % CH, grow = row - lane + rr;
        const uint4 val = *reinterpret_cast<const uint4*>(stg + rr * (HD * 2) + ((c ^ (rr % CH)) << 4));
        if (grow < N) reinterpret_cast<uint4*>(args.o + (((size_t)b * N + grow) * args.Hq + h) * HD)[c] = val;
      }
      if (row_ok) args.lse[((size_t)b * args.Hq + h) * N + row] = m + logf(l);
    } else if (row_ok) {
      const float f = A / l;
      __half* orow = args.o + (((size_t)b * N + row) * args.Hq + h) * HD + hc * OW;
#pragma unroll
      for (int c = 0; c < OW / 8; ++c) {
        __half2 hv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) hv[e] = __floats2half2_rn(O[c * 8 + 2 * e] * f, O[c * 8 + 2 * e + 1] * f);
        reinterpret_cast<uint4*>(orow)[c] = *reinterpret_cast<uint4*>(hv);
      }
      if (hc == 0) args.lse[((size_t)b * args.Hq + h) * N + row] = m + logf(l);
    }
    PROF_T(epi1);
    PROF_ADD(8, epi0, epi1);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
#ifdef TURBO_PROFILE
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int i = 0; i < 17; ++i)
      if (prof_acc[i]) atomicAdd(&g_prof[i], (unsigned long long)prof_acc[i]);
  if (threadIdx.x == 0) {
    atomicAdd(&g_prof[20], (unsigned long long)nkv);
    atomicAdd(&g_prof[21], 1ull);
    atomicAdd(&g_prof[22], (unsigned long long)(clock64() - t_cta0));
  }
#endif
}

}  // namespace ta

// ---------------------------------------------------------------------------
namespace ta_host {
using namespace ta;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess) return nullptr;
  return reinterpret_cast<EncodeTiledFn>(fn);
}

static bool make_map_3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                        uint64_t s2, uint32_t b0, uint32_t b1, CUtensorMapSwizzle swz,
                        CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_UINT8) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1, s2};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

#ifdef TURBO_PROFILE
extern "C" TURBO_API void turbo_debug_prof(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_prof, sizeof(g_prof));
  if (reset) {
    unsigned long long z[32] = {0};
    cudaMemcpyToSymbol(g_prof, z, sizeof(z));
  }
}
#endif

cudaError_t launch_prefill(const turbo_params_t* p, int B, int N, int Nk, int Hq, int Hkv, int causal, const __half* q,
                           const int8_t* k1, const __half* v1t, const float* k1s, const float* v1s, __half* o,
                           float* lse, cudaStream_t st) {
  const int HD = p->head_dim, Tc = (Nk + kBc - 1) / kBc;
  CUtensorMap tmk, tmv;
  const CUtensorMapSwizzle swk = HD == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  if (!make_map_3d(&tmk, k1, HD, Nk, (uint64_t)B * Hkv, HD, (uint64_t)Nk * HD, HD, kBc, swk))
    return cudaErrorInvalidValue;
  if (!make_map_3d(&tmv, v1t, kBc, HD, (uint64_t)B * Hkv * Tc, kBc * 2, (uint64_t)HD * kBc * 2, kBc, HD,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_FLOAT16))
    return cudaErrorInvalidValue;
  PrefillArgs a;
  a.q = q;
  a.o = o;
  a.lse = lse;
  a.k1s = k1s;
  a.v1s = v1s;
  a.B = B;
  a.N = N;
  a.Nk = Nk;
  a.q0 = Nk - N;
  a.Hq = Hq;
  a.Hkv = Hkv;
  a.causal = causal;
  a.block_q = p->block_q;
  a.alpha_mode = p->alpha_mode;
  const int G = Hq / Hkv;
  const bool pair = (G % 2) == 0;  // slots = two heads of a GQA group, else two adjacent query tiles
  a.n_qtiles = (N + kTileM - 1) / kTileM;
  if (!pair) a.n_qtiles = (a.n_qtiles + 1) / 2;
  a.scale = p->softmax_scale;
  fill_sas_const(&a.sas, p->sas_nr);
  a.has_tap = p->debug_tap != nullptr;
  if (a.has_tap) a.tap = *reinterpret_cast<const turbo_debug_tap_t*>(p->debug_tap);
  else memset(&a.tap, 0, sizeof(a.tap));
  const dim3 grid((unsigned)(a.n_qtiles * B * Hq / (pair ? 2 : 1)));
  {
    const int GS = G / (pair ? 2 : 1), units = B * Hkv * GS;
    int ug = GS * std::max(1, (4 * 148 + a.n_qtiles * GS - 1) / (a.n_qtiles * GS));
    a.unit_group = std::min(units, ug);
  }
#define TA_LAUNCH_T(HDV, NSV, SPV, TAPV, TPV)                                                                  \
  {                                                                                                        \
    const size_t smem = sizeof(PrefillSmem<HDV, NSV, SPV>) + 1024;                                         \
    cudaFuncSetAttribute(prefill_kernel<HDV, NSV, SPV, TAPV, TPV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         (int)smem);                                                                       \
    prefill_kernel<HDV, NSV, SPV, TAPV, TPV><<<grid, 128 * (1 + NSV * SPV), smem, st>>>(tmk, tmv, a);           \
  }
#define TA_LAUNCH_P(HDV, NSV, SPV, TAPV) \
  if (pair) TA_LAUNCH_T(HDV, NSV, SPV, TAPV, false) else TA_LAUNCH_T(HDV, NSV, SPV, TAPV, true)
#define TA_LAUNCH(HDV, NSV, SPV) \
  if (a.has_tap) TA_LAUNCH_P(HDV, NSV, SPV, true) else TA_LAUNCH_P(HDV, NSV, SPV, false)
  if (HD == 128) TA_LAUNCH(128, 2, TA_PREFILL_SPLIT) else TA_LAUNCH(64, 2, TA_PREFILL_SPLIT)
#undef TA_LAUNCH
#undef TA_LAUNCH_P
#undef TA_LAUNCH_T
  return cudaGetLastError();
}
}  // namespace ta_host
