// prefill.cu -- Algorithm 1 (TurboAttention prefill) on sm_100a.
//
// One CTA = one (batch, pair of GQA query heads sharing a KV head, 128-row
// query tile) -- or, for odd G, two adjacent 128-row tiles of one head; each
// tile ("slot") holds two B_r = 64 quantisation blocks (or one B_r = 128 block).
// One CTA per SM (all 512 TMEM columns: per slot S_0 | S_1 | O).  Warp roles:
//   warp 0      TMA producer: K_j [64 x d] and V_j^T [d x 64] tiles of stage-1 codes
//               carried exactly in FP16, into a 3-stage smem ring shared by both slots.
//   warps 1, 2  one single-thread tcgen05.mma issuer per slot (warp 1 also owns
//               TMEM): S_j = Q^q1 K_j^q1^T (kind::f16 on the integer codes: every
//               product and partial sum is an integer below 2^24, so the fp32
//               accumulator holds S_int exactly and pass 1 needs no int->float
//               conversion; double-buffered) and
//               O^ += P'_j V_j^q1 (kind::f16, A = P' from TMEM, B = V codes from
//               smem, fp32 accumulator in TMEM across all key tiles).
//   warps 4-11  one softmax warpgroup per slot, thread = query row = TMEM lane:
//               Q stage-1 quantisation (prologue); per key tile, S_j -> registers
//               (one TMEM round trip), x, row max, SAS (LUT x POLY), row sum, P
//               scale and codes -- all register-resident -- then P' = Pc s_P s_V R
//               as an exact fp16 hi + lo pair written over S_j's columns (the A
//               operand of the two P.V MMAs); epilogue O = O^ / (R l).
//
// Scaled output accumulator (tolerance set, R-16): O_true = O^ / R per row, with
// R_j = R_{j-1} / alpha_j, so tile j's alpha never touches O^ (P:921 rescale folded
// into R).  F = s_P s_V R is kept in [2^-14, 60] by exact power-of-two rescales of
// the row of O^ (rare); alpha = 0 restarts the row.  P' = Pc F with F = F_hi + F_lo,
// F_hi = F rounded to 4 significant bits, so Pc F_hi (<= 11 bits) is exact in fp16
// and only Pc F_lo is rounded: P' carries a relative error <= 2^-15 (the running O
// of round 1 accumulated in fp32 registers).
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace ta {

constexpr int kTileM = 128;
constexpr int kSlotCols = 256;  // per slot: S [0,128) (B_c = 64: S_0 [0,64) S_1 [64,128)) O [128, 128 + d)
// K/V ring depth: 3 stages of 24 KB (B_c = 64), 2 stages of 48 KB (B_c = 128; 227 KB of smem)
template <int BC>
constexpr int stages_of() { return BC == 64 ? 3 : 2; }

template <int HD, int BC>
struct PrefillSmem {
  static constexpr int kStages = stages_of<BC>();
  // Q^q1 codes as fp16 (exact), K-major SW128: HD / 64 atoms of [128 rows][64 channels] (128-B rows).  Once
  // the slot's last QK^T MMA has completed, its buffer stages the epilogue's O rows.
  __half q1[2][kTileM * HD];
  __half k[kStages][BC * HD];  // K_j^q1 codes as fp16, HD / 64 atoms of [B_c keys][64 channels] (SW128)
  __half v[kStages][HD * BC];  // V_j^q1 codes as fp16, transposed, B_c / 64 tiles [HD][64] (128-B rows, SW128)
  uint64_t kv_full[kStages], kv_empty[kStages];
  uint64_t s_full[2][2], p_full[2][2], pv_done[2], q_ready;
  uint32_t tmem_base;
  float red_a[2][4];
  float red_p[2][2][4];  // [slot][tile parity][quadrant] warp P maxima
};

struct PrefillArgs {
  const __half* q;
  const int8_t* q1_in;  // pre-quantised Q^q1 [B][N][Hq][d] (turbo_q_projection) or NULL
  const float* sq_in;   // its scales [B][Hq][ceil(N / B_r)]
  __half* o;
  float* lse;
  const float* k1s;
  const float* v1s;
  int B, N, Hq, Hkv, causal, block_q, alpha_mode, n_qtiles, unit_group, scale_fp16;
  int q_prefetch;  // > 0: warp 3 prefetches into L2 the FP16 Q rows of CTA blockIdx.x + q_prefetch (a wave later)
  int Nk, q0;  // keys per sequence; absolute position of query row 0 (chunked prefill: Nk - N)
  float scale;
  SasConst sas;
  int has_tap;
  turbo_debug_tap_t tap;
};

// Byte offset of the 16-byte chunk c8 (channels 8 c8 .. 8 c8 + 7, fp16) of row r in a K-major SW128
// operand of `rows` rows split into 64-channel atoms of 128-B rows.
TA_DEV uint32_t f16_swz(int rows, int r, int c8) {
  return (uint32_t)((c8 >> 3) * rows * 128 + r * 128 + (((c8 & 7) ^ (r & 7)) << 4));
}
// fp16 pair of two stage-1 codes given as magic-float bits (rint_prod_bits: magic + code, exact)
TA_DEV uint32_t codes_h2(uint32_t b0, uint32_t b1) {
  const __half2 h = __floats2half2_rn(__uint_as_float(b0) - kMagic, __uint_as_float(b1) - kMagic);
  return *reinterpret_cast<const uint32_t*>(&h);
}
// fp16 pairs of the four signed bytes of w (exact)
TA_DEV void bytes_h2(uint32_t w, uint32_t& lo, uint32_t& hi) {
  const __half2 a = __floats2half2_rn((float)(int8_t)(w & 0xFF), (float)(int8_t)((w >> 8) & 0xFF));
  const __half2 b = __floats2half2_rn((float)(int8_t)((w >> 16) & 0xFF), (float)(int8_t)(w >> 24));
  lo = *reinterpret_cast<const uint32_t*>(&a);
  hi = *reinterpret_cast<const uint32_t*>(&b);
}


// Window of F = s_P s_V R outside which the row of O^ is rescaled by a power of two.
// Upper: fp16(-1024 F_hi) must be finite (F_hi <= 63.97) for the P' hi/lo split.
// Lower: F_hi must be a normal fp16 (>= 2^-14) so that P c F_hi stays exact; below
// 2^-9 the lo part is subnormal, an absolute error <= 2^-25 per P' element against
// a row whose largest tile has F >= 1 (the first visible tile sets F in [1, 2)).
constexpr float kFmax = 60.f;
constexpr float kFmin = 0.00006103515625f;  // 2^-14

// F = 2^e m, m in [1, 2): 2^-e (exact power of two; F normal and positive)
TA_DEV float inv_pow2_of(float F) { return __uint_as_float((uint32_t)(254 - (__float_as_uint(F) >> 23)) << 23); }

template <int HD, bool TAP, bool TP, bool PROW, int BC, bool SF>
__global__ void __launch_bounds__(384, 1)
    prefill_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                   const __grid_constant__ PrefillArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  using Smem = PrefillSmem<HD, BC>;
  constexpr int kStages = Smem::kStages;
  // 1024-B aligned (128B-swizzle atoms); pointer arithmetic keeps the shared address space.
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // Work item: (query tile, batch, kv head, head pair).  Units are taken in groups of
  // UG (about 4 x 148 CTAs' worth), heaviest (last) query tiles first inside a group
  // for causal load balance; the group keeps the K/V streams resident in L2.
  const int G = args.Hq / args.Hkv, GS = TP ? G : G / 2;
  const int units = args.B * args.Hkv * GS;
  const int UG = args.unit_group;
  // (query tile, batch, kv head, head group) of CTA number cta
  auto unit_of = [&](int cta, int& it_, int& b_, int& kvh_, int& hg_) {
    const int gi = cta / (UG * args.n_qtiles), rm = cta % (UG * args.n_qtiles);
    const int ug = min(UG, units - gi * UG);
    it_ = args.n_qtiles - 1 - rm / ug;
    const int uu = gi * UG + rm % ug;
    b_ = uu / (args.Hkv * GS);
    kvh_ = (uu / GS) % args.Hkv;
    hg_ = uu % GS;
  };
  int it, b, kvh, hg;
  unit_of((int)blockIdx.x, it, b, kvh, hg);
  const int h0 = kvh * G + hg * (TP ? 1 : 2);
  const int N = args.N, Tc = (args.Nk + BC - 1) / BC;  // N query rows, Tc key tiles (B_c keys each)
  auto tile_of = [&](int s) { return TP ? 2 * it + s : it; };
  auto nkv_of = [&](int s) {
    const int ti = tile_of(s);
    if (ti * kTileM >= N) return 0;
    const int last_row = min(ti * kTileM + kTileM - 1, N - 1);
    return args.causal ? min(Tc, (args.q0 + last_row) / BC + 1) : Tc;
  };
  const int nkv = max(nkv_of(0), nkv_of(1));  // key tiles the CTA streams (both slots walk all of them)
  const size_t bkv = (size_t)b * args.Hkv + kvh;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.kv_full[s], 1);
      mbar_init(&sm.kv_empty[s], 2);  // one commit per MMA issuer
    }
    for (int t = 0; t < 2; ++t) {
      for (int s = 0; s < 2; ++s) {
        mbar_init(&sm.s_full[t][s], 1);
        mbar_init(&sm.p_full[t][s], 4);  // one arrival per softmax warp
      }
      mbar_init(&sm.pv_done[t], 1);
    }
    mbar_init(&sm.q_ready, 256);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&sm.tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");  // 384 thr x 168 -> 128 x 56 + 256 x 224
    if (warp == 0) {
      // ---------------------------------------------------------- TMA producer
      if (elect_one()) {
        tma_prefetch_desc(&tm_k);
        tma_prefetch_desc(&tm_v);
        for (int j = 0; j < nkv; ++j) {
          const int st = j % kStages, n = j / kStages;
          if (n > 0) mbar_wait(&sm.kv_empty[st], (n - 1) & 1);
          mbar_expect_tx(&sm.kv_full[st], 4 * BC * HD);  // K and V fp16
#pragma unroll
          for (int a = 0; a < HD / 64; ++a)  // K^T: one [B_c][64] fp16 box per 64 channels
            tma_load_3d(sm.k[st] + a * BC * 64, &tm_k, &sm.kv_full[st], 64 * a, j * BC, (int)bkv);
#pragma unroll
          for (int u = 0; u < BC / 64; ++u)  // V^T: one [HD][64] box per 64 keys
            tma_load_3d(sm.v[st] + u * HD * 64, &tm_v, &sm.kv_full[st], 64 * u, 0, (int)(bkv * Tc + j));
        }
      }
    } else if (warp == 3) {
      // ---------------------------------------------------------- Q prefetch (otherwise idle warp)
      // The FP16 Q rows (2 x 128 rows of 2 d bytes) of the CTA that starts about a wave later go to L2 now,
      // so that CTA's prologue loads hit L2 instead of waiting on HBM.
      const int nxt = (int)blockIdx.x + args.q_prefetch;
      if (args.q_prefetch > 0 && args.q1_in == nullptr && nxt < (int)gridDim.x) {
        int it2, b2, kvh2, hg2;
        unit_of(nxt, it2, b2, kvh2, hg2);
        const int hb = kvh2 * G + hg2 * (TP ? 1 : 2);
        for (int i = lane; i < 2 * kTileM; i += 32) {
          const int s2 = i / kTileM, rr = i % kTileM;
          const int row2 = (TP ? 2 * it2 + s2 : it2) * kTileM + rr, h2 = TP ? hb : hb + s2;
          if (row2 < N)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                             args.q + (((size_t)b2 * N + row2) * args.Hq + h2) * HD),
                         "r"(HD * 2)
                         : "memory");
        }
      }
    } else if (warp == 1 || warp == 2) {
      // ---------------------------------------------------------- MMA issuers (one per slot)
      // Issue order S_0, S_1, PV_0, S_2, PV_1, ...: S_{j+1} lands in the TMEM columns of
      // P'_{j-1}, which PV_{j-1} (issued before it) has consumed -- tcgen05.mma of one
      // thread executes in order.
      const int t = warp - 1;
      constexpr uint32_t idesc_qk = idesc_f16(kTileM, BC);  // fp16 codes, fp32 S: exact integers
      constexpr uint32_t idesc_pv = idesc_f16(kTileM, HD);
      const uint32_t tslot = tmem + t * kSlotCols;
      mbar_wait(&sm.q_ready, 0);
      tc_fence_after();
      // B_c = 64: S double-buffered (S_{j+1} issued before PV_j).  B_c = 128: S_j takes all
      // 128 columns, so S_{j+1} follows PV_j (lag 0).
      constexpr int kLag = BC == 64 ? 1 : 0;
      for (int j = 0; j < nkv + kLag; ++j) {
        if (j < nkv) {
          const int st = j % kStages, sb = BC == 64 ? (j & 1) : 0;
          mbar_wait(&sm.kv_full[st], (j / kStages) & 1);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t q1a = smem_u32(sm.q1[t]), ka = smem_u32(sm.k[st]);
#pragma unroll
            for (int ks = 0; ks < HD / 16; ++ks)  // K = 16 channels: atom ks / 4, 32 B into its 128-B rows
              mma_f16_ss(tslot + sb * 64, smem_desc(q1a + (ks >> 2) * kTileM * 128 + (ks & 3) * 32, 1024, kSw128),
                         smem_desc(ka + (ks >> 2) * BC * 128 + (ks & 3) * 32, 1024, kSw128), idesc_qk, ks > 0);
            mma_commit(&sm.s_full[t][sb]);
          }
          __syncwarp();
        }
        if (j >= kLag) {
          const int jj = j - kLag, pb = BC == 64 ? (jj & 1) : 0, st = jj % kStages;
          mbar_wait(&sm.p_full[t][pb], BC == 64 ? ((jj >> 1) & 1) : (jj & 1));
          tc_fence_after();
          if (elect_one()) {
            const uint32_t va = smem_u32(sm.v[st]);
#pragma unroll
            for (int u = 0; u < BC / 64; ++u)  // 64-key sub-tiles: P' in columns [64u, 64u + 64)
#pragma unroll
              for (int part = 0; part < 2; ++part)  // P'_hi, then P'_lo (32 columns each)
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                  mma_f16_ts(tslot + 128, tslot + (pb + u) * 64 + part * 32 + ks * 8,
                             smem_desc(va + u * HD * 128 + ks * 32, 1024, kSw128), idesc_pv,
                             (jj | u | part | ks) != 0);
            mma_commit(&sm.pv_done[t]);
            mma_commit(&sm.kv_empty[st]);
          }
          __syncwarp();
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
    // ------------------------------------------------------------ softmax
    const int widx = warp - 4, slot = widx >> 2, h = TP ? h0 : h0 + slot;
    const int its = tile_of(slot);
    const int qd = warp & 3, r = qd * 32 + lane, row = its * kTileM + r;
    const bool row_ok = row < N;
    const int half = args.block_q == 64 ? (r >> 6) : 0;  // P-scale group (B_r rows)
    const uint32_t tbase = tmem + ((uint32_t)(qd * 32) << 16) + slot * kSlotCols;
    const float lut_lane = sas_lut_lane(args.sas, lane);
    const float nr_abs = args.sas.nr_abs;
    const float p_top = sas_eval_v<SF>(0.f, lut_lane, nr_abs);  // SAS(0): the largest possible P~
    const float inv_top = div_119_by(p_top), s_top = div_by_119(p_top);
    const bool tap_cta = TAP && args.tap.batch == b && args.tap.head == h && (args.tap.i_block >> 1) == its;
    const bool tap_row = tap_cta && (args.tap.i_block & 1) == (r >> 6);
    const uint32_t bar_slot = 1 + slot;                                  // the slot's 128 threads
    // the P-scale group's two named barriers (alternating by tile parity: a warp that only arrives may
    // reach the next tile's exchange before its partner has waited on this one)
    const uint32_t bar_grp = args.block_q == 64 ? 3 + (slot * 2 + half) * 2 : 11 + slot * 2;
    const uint32_t grp_threads = args.block_q;

    // Q stage-1 quantisation (Alg. 1; per B_r x d block) -- or, with q1_in, the codes and
    // scales the Q projection's epilogue produced (turbo_q_projection)
    float s_q;
    if (args.q1_in) {
      const int nbq = (N + args.block_q - 1) / args.block_q;
      s_q = row_ok ? args.sq_in[((size_t)b * args.Hq + h) * nbq + row / args.block_q] : 0.f;
      const uint4* src = reinterpret_cast<const uint4*>(args.q1_in + (((size_t)b * N + row) * args.Hq + h) * HD);
#pragma unroll
      for (int c = 0; c < HD / 16; ++c) {
        const uint4 w = row_ok ? src[c] : make_uint4(0, 0, 0, 0);
        uint32_t h[8];
        bytes_h2(w.x, h[0], h[1]);
        bytes_h2(w.y, h[2], h[3]);
        bytes_h2(w.z, h[4], h[5]);
        bytes_h2(w.w, h[6], h[7]);
        uint8_t* qb = reinterpret_cast<uint8_t*>(sm.q1[slot]);
        *reinterpret_cast<uint4*>(qb + f16_swz(kTileM, r, 2 * c)) = make_uint4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<uint4*>(qb + f16_swz(kTileM, r, 2 * c + 1)) = make_uint4(h[4], h[5], h[6], h[7]);
        if (tap_row) *reinterpret_cast<uint4*>(args.tap.q1 + (r & 63) * HD + c * 16) = w;
      }
      if (tap_row && (r & 63) == 0) args.tap.s_q[0] = s_q;
    } else {
      uint4 qraw[HD / 8];
      float qa = 0.f;
      const __half* qrow = args.q + (((size_t)b * N + row) * args.Hq + h) * HD;
#pragma unroll
      for (int c = 0; c < HD / 8; ++c) {
        qraw[c] = row_ok ? reinterpret_cast<const uint4*>(qrow)[c] : make_uint4(0, 0, 0, 0);
        const __half2* hp = reinterpret_cast<const __half2*>(&qraw[c]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 f = __half22float2(hp[e]);
          qa = fmaxf(qa, fmaxf(fabsf(f.x), fabsf(f.y)));
        }
      }
      qa = warp_max_nonneg(qa);
      if (lane == 0) sm.red_a[slot][qd] = qa;
      named_bar_sync(bar_slot, 128);
      const float a_q = args.block_q == 64 ? fmaxf(sm.red_a[slot][2 * half], sm.red_a[slot][2 * half + 1])
                                           : fmaxf(fmaxf(sm.red_a[slot][0], sm.red_a[slot][1]),
                                                   fmaxf(sm.red_a[slot][2], sm.red_a[slot][3]));
      const float inv_q = a_q > 0.f ? div_119_by(a_q) : 0.f;
      s_q = st1_scale(div_by_119(a_q), args.scale_fp16);  // (FP16 variant: R-29)
#pragma unroll
      for (int c = 0; c < HD / 8; ++c) {  // 8 channels: one 16-B chunk of fp16 codes
        const __half2* hp = reinterpret_cast<const __half2*>(&qraw[c]);
        uint32_t bq[8], h[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __half22float2(hp[e]);
          bq[2 * e] = rint_prod_bits(f.x, inv_q);
          bq[2 * e + 1] = rint_prod_bits(f.y, inv_q);
          h[e] = codes_h2(bq[2 * e], bq[2 * e + 1]);
        }
        *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(sm.q1[slot]) + f16_swz(kTileM, r, c)) =
            make_uint4(h[0], h[1], h[2], h[3]);
        if (tap_row)
          *reinterpret_cast<uint2*>(args.tap.q1 + (r & 63) * HD + c * 8) =
              make_uint2(pack4_lo(bq[0], bq[1], bq[2], bq[3]), pack4_lo(bq[4], bq[5], bq[6], bq[7]));
      }
      if (tap_row && (r & 63) == 0) args.tap.s_q[0] = s_q;
    }
    fence_proxy_async();
    mbar_arrive(&sm.q_ready);

    float m = -INFINITY, l = 0.f, R = 0.f;  // O_true = O^ / R (R = 0: nothing accumulated yet)
    const int kmax = row_ok ? (args.causal ? args.q0 + row : args.Nk - 1) : -1;  // last visible key of this row
    const int tap_j = TAP ? args.tap.j_block : -2;

    for (int j = 0; j < nkv; ++j) {
      const int sb = BC == 64 ? (j & 1) : 0, rb = j & 1;  // S buffer; P-max exchange parity
      const uint32_t tS = tbase + sb * 64;
      mbar_wait_spin(&sm.s_full[slot][sb], BC == 64 ? ((j >> 1) & 1) : (j & 1));
      tc_fence_after();
      const int nvalid = max(0, min(BC, kmax - j * BC + 1));  // visible keys of the tile
      const bool active = nvalid > 0;
      const bool full = __all_sync(0xffffffffu, nvalid == BC);
      uint32_t v[BC];
#pragma unroll
      for (int c = 0; c < BC; c += 32) TA_TMEM_LD32(tS + c, (v + c));
      tmem_ld_wait();
      if (TAP && tap_row && j == tap_j)
        for (int c = 0; c < BC; ++c) args.tap.s_int[(r & 63) * BC + c] = c < nvalid ? (int)__uint_as_float(v[c]) : 0;
      // x = S s_Q s_K / sqrt(d) (R-18); masked keys -> -inf
      const float cqk = __fmul_rn(__fmul_rn(s_q, args.k1s[bkv * Tc + j]), args.scale);
      const float s_v = args.v1s[bkv * Tc + j];
      float mt = -INFINITY, mt1 = -INFINITY;
      {
        const f32x2 cq2 = pk2(cqk, cqk);
        if (full) {
#pragma unroll
          for (int c = 0; c < BC; c += 4) {  // two independent max chains
            const f32x2 x2 = mul2(pk2(__uint_as_float(v[c]), __uint_as_float(v[c + 1])), cq2);  // S: exact fp32
            const f32x2 y2 = mul2(pk2(__uint_as_float(v[c + 2]), __uint_as_float(v[c + 3])), cq2);
            mt = fmaxf(mt, fmaxf(lo2(x2), hi2(x2)));
            mt1 = fmaxf(mt1, fmaxf(lo2(y2), hi2(y2)));
            v[c] = __float_as_uint(lo2(x2));
            v[c + 1] = __float_as_uint(hi2(x2));
            v[c + 2] = __float_as_uint(lo2(y2));
            v[c + 3] = __float_as_uint(hi2(y2));
          }
        } else {
#pragma unroll
          for (int c = 0; c < BC; c += 2) {
            const f32x2 x2 = mul2(pk2(__uint_as_float(v[c]), __uint_as_float(v[c + 1])), cq2);
            const float x0 = c < nvalid ? lo2(x2) : -INFINITY;
            const float x1 = c + 1 < nvalid ? hi2(x2) : -INFINITY;
            mt = fmaxf(mt, fmaxf(x0, x1));
            v[c] = __float_as_uint(x0);
            v[c + 1] = __float_as_uint(x1);
          }
        }
        mt = fmaxf(mt, mt1);
      }
      // m_new, alpha = SAS(m_prev - m_new) (R-15)
      const float m_new = fmaxf(m, mt);
      float alpha = sas_eval_v<SF>(__fsub_rn(m_new, m), lut_lane, nr_abs);
      if (m == -INFINITY) alpha = 0.f;
      else if (args.alpha_mode == 1 && m_new == m) alpha = 1.f;
      const float m_use = active ? m_new : 0.f;  // inactive row: every x = -inf -> P~ = 0
      // P~ = SAS(x - m_new) in registers; two elements per FADD2 / FFMA2 / FMUL2,
      // bit-identical to the scalar sas_eval.
      float pmax = 0.f, pmax1 = 0.f;
      f32x2 rsum2;
      f32x2 rs[4] = {pk2(0.f, 0.f), pk2(0.f, 0.f), pk2(0.f, 0.f), pk2(0.f, 0.f)};  // 4 row-sum chains
      {
        const f32x2 m2 = pk2(m_use, m_use), mg2 = pk2(kMagic, kMagic);
        const f32x2 c3 = pk2(-0.1025f, -0.1025f), c2 = pk2(0.4626f, 0.4626f), c1 = pk2(-0.9922f, -0.9922f),
                    c0 = pk2(0.9996f, 0.9996f);
#pragma unroll
        for (int c = 0; c < BC; c += 2) {
          const f32x2 d2 = sub2(m2, pk2(__uint_as_float(v[c]), __uint_as_float(v[c + 1])));
          const f32x2 t2 = add2_rd(d2, mg2);         // kMagic + floor(d)
          const f32x2 f2 = sub2(d2, sub2(t2, mg2));  // d - floor(d), exact
          const float l0 = lut_shfl(lut_lane, __float_as_uint(lo2(t2)));
          const float l1 = lut_shfl(lut_lane, __float_as_uint(hi2(t2)));
          const f32x2 p2 = SF ? sas_poly2_h(f2) : fma2(fma2(fma2(c3, f2, c2), f2, c1), f2, c0);  // R-30 / R-13
          const f32x2 lp = mul2(pk2(l0, l1), p2);
          const float pt0 = lo2(d2) > nr_abs ? 0.f : lo2(lp);
          const float pt1 = hi2(d2) > nr_abs ? 0.f : hi2(lp);
          rs[(c >> 1) & 3] = add2(rs[(c >> 1) & 3], pk2(pt0, pt1));
          if (c & 2) pmax1 = fmaxf(pmax1, fmaxf(pt0, pt1));  // two independent max chains
          else pmax = fmaxf(pmax, fmaxf(pt0, pt1));
          v[c] = __float_as_uint(pt0);
          v[c + 1] = __float_as_uint(pt1);
        }
        rsum2 = add2(add2(rs[0], rs[1]), add2(rs[2], rs[3]));
        pmax = fmaxf(pmax, pmax1);
      }
      const float m_prev = m;
      if (active) {
        l = alpha * l + (lo2(rsum2) + hi2(rsum2));  // l = SAS(m_prev - m_new) l + rowsum(P~)
        m = m_new;
      }
      // P scale: max P~ over the B_r x B_c tile (or, PROW, over the row)
      float a_p = pmax;
      if (!PROW) {
        // Every P~ <= SAS(0) (LUT <= 1, POLY decreasing on [0, 1], the rounding of c0 - |.| f never
        // exceeds c0), so a warp whose maximum is SAS(0) knows the tile's maximum: it publishes and only
        // arrives; warps without it publish, wait and combine.
        const float wmax = warp_max_nonneg(pmax);
        if (lane == 0) sm.red_p[slot][rb][qd] = wmax;
        if (wmax == p_top) {
          named_bar_arrive(bar_grp + rb, grp_threads);
          a_p = p_top;
        } else {
          named_bar_sync(bar_grp + rb, grp_threads);
          a_p = args.block_q == 64 ? fmaxf(sm.red_p[slot][rb][2 * half], sm.red_p[slot][rb][2 * half + 1])
                                   : fmaxf(fmaxf(sm.red_p[slot][rb][0], sm.red_p[slot][rb][1]),
                                           fmaxf(sm.red_p[slot][rb][2], sm.red_p[slot][rb][3]));
        }
      }
      float inv_p = inv_top, s_p = s_top;  // the common case a_P = SAS(0): its scale and reciprocal, once
      if (a_p != p_top) {
        inv_p = a_p > 0.f ? div_119_by(a_p) : 0.f;
        s_p = div_by_119(a_p);
      }
      // Scale bookkeeping: O^ row *= fix (fix = 0: alpha = 0 discards the history;
      // power of two: keeps F = s_P s_V R in [2^-8, 2^5]).
      float F = 0.f, fix = 1.f;
      if (active) {
        if (m_prev != -INFINITY && alpha == 0.f) {
          fix = 0.f;
          R = 0.f;
        } else if (R != 0.f) {
          R = alpha == 1.f ? R : __fdividef(R, alpha);
        }
        const float sps = __fmul_rn(s_p, s_v);
        if (R == 0.f && sps > 0.f) R = inv_pow2_of(sps);  // first contribution: F in [1, 2)
        F = __fmul_rn(sps, R);
        if (F > kFmax || (F > 0.f && F < kFmin)) {
          const float f = inv_pow2_of(F);
          R *= f;
          F *= f;
          fix *= f;
        }
      }
      if (TAP && tap_row && j == tap_j) {  // tapped tile: O^ <- PV_int exactly (P' = Pc)
        fix = 0.f;
        F = 1.f;
      }
      // O^ is quiescent once PV_{j-1} is done.  Only a rescale (or the tap) touches O^ here; at B_c = 128 the
      // wait is skipped otherwise: S_j's s_full commit already covers PV_{j-1} there (S_j is issued after it),
      // so pv_done is never behind the phase awaited next (j' - 1, or nkv - 1 in the epilogue): +4.6 %.  At
      // B_c = 64 (S_j issued after PV_{j-2} only) the per-tile wait is kept -- skipping it measured 1.1 % slower.
      const bool rescale = __any_sync(0xffffffffu, fix != 1.f);
      if (j >= 1 && (BC == 64 || rescale || j == nkv - 1 || (TAP && __any_sync(0xffffffffu, tap_row && j - 1 == tap_j)))) {
        mbar_wait_spin(&sm.pv_done[slot], (j - 1) & 1);
        tc_fence_after();
        if (TAP && tap_row && j - 1 == tap_j) {
#pragma unroll 1
          for (int cc = 0; cc < HD / 32; ++cc) {
            uint32_t o[32];
            TA_TMEM_LD32(tbase + 128 + cc * 32, o);
            tmem_ld_wait();
            for (int e = 0; e < 32; ++e) args.tap.pv_int[(r & 63) * HD + cc * 32 + e] = (int)__uint_as_float(o[e]);
          }
        }
      }
      if (rescale) {  // rare: rescale / restart this warp's O^ rows
#pragma unroll 1
        for (int cc = 0; cc < HD / 32; ++cc) {
          uint32_t o[32];
          TA_TMEM_LD32(tbase + 128 + cc * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * fix);
          TA_TMEM_ST32(tbase + 128 + cc * 32, o);
        }
        tmem_st_wait();
      }
      // P codes Pc = rne(P~ 119 / a_P) (R-27) and P' = Pc F_hi + Pc F_lo as fp16
      {
        const float Fh = __uint_as_float((__float_as_uint(F) + 0x80000u) & 0xFFF00000u);
        const __half fh = __float2half_rn(Fh), fl = __float2half_rn(__fsub_rn(F, Fh));
        const __half nfh = __float2half_rn(-1024.f * Fh), nfl = __float2half_rn(-1024.f * __half2float(fl));
        const uint32_t fh2 = (uint32_t)__half_as_ushort(fh) * 0x10001u, fl2 = (uint32_t)__half_as_ushort(fl) * 0x10001u;
        const uint32_t nfh2 = (uint32_t)__half_as_ushort(nfh) * 0x10001u,
                       nfl2 = (uint32_t)__half_as_ushort(nfl) * 0x10001u;
        constexpr float kMagicF16 = 12582912.0f + 25600.0f;  // 1.5*2^23 + 0x6400: low half = fp16(1024 + code)
        const f32x2 inv2 = pk2(inv_p, inv_p), mf2 = pk2(kMagicF16, kMagicF16);
#pragma unroll
        for (int u = 0; u < BC / 64; ++u) {  // per 64 keys: P'_hi in columns [64u, 64u + 32), P'_lo after it
          uint32_t y[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const int c = 64 * u + 2 * e;
            const f32x2 y2 = fma2(pk2(__uint_as_float(v[c]), __uint_as_float(v[c + 1])), inv2, mf2);
            if (TAP && tap_row && j == tap_j) {
              args.tap.p_codes[(r & 63) * BC + c] = (uint8_t)__float_as_uint(lo2(y2));
              args.tap.p_codes[(r & 63) * BC + c + 1] = (uint8_t)__float_as_uint(hi2(y2));
            }
            y[e] = __byte_perm(__float_as_uint(lo2(y2)), __float_as_uint(hi2(y2)), 0x5410);
          }
          uint32_t ph[32], pl[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) ph[e] = hfma2_u32(y[e], fh2, nfh2);  // Pc F_hi, exact
          TA_TMEM_ST32(tS + 64 * u, ph);
#pragma unroll
          for (int e = 0; e < 32; ++e) pl[e] = hfma2_u32(y[e], fl2, nfl2);  // Pc F_lo, one rounding
          TA_TMEM_ST32(tS + 64 * u + 32, pl);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();  // every lane's P' stores precede the warp's single arrival
      if (lane == 0) mbar_arrive(&sm.p_full[slot][sb]);
      if (TAP && tap_row && j == tap_j) {
        args.tap.m_new[r & 63] = m;
        if ((r & 63) == 0) args.tap.s_p[0] = s_p;
      }
    }
    // Epilogue: O_i = diag(l)^-1 O with O = O^ / R; L_i = m + log l
    mbar_wait_spin(&sm.pv_done[slot], (nkv - 1) & 1);
    tc_fence_after();
    if (TAP && tap_row && nkv - 1 == tap_j) {
#pragma unroll 1
      for (int cc = 0; cc < HD / 32; ++cc) {
        uint32_t o[32];
        TA_TMEM_LD32(tbase + 128 + cc * 32, o);
        tmem_ld_wait();
        for (int e = 0; e < 32; ++e) args.tap.pv_int[(r & 63) * HD + cc * 32 + e] = (int)__uint_as_float(o[e]);
      }
    }
    {
      // O rows go through shared memory (this warp's 32 rows, XOR-swizzled 16-byte chunks)
      // so that the global stores are row-contiguous.
      constexpr int CH = HD / 8;  // 16-byte chunks per row
      // (the slot's Q buffer: its last QK^T MMA completed before the last tile's S was read)
      uint8_t* stg = reinterpret_cast<uint8_t*>(sm.q1[slot]) + qd * (32 * HD * 2);
      const float f = (row_ok && R > 0.f) ? 1.f / (R * l) : 0.f;
#pragma unroll
      for (int cc = 0; cc < HD / 32; ++cc) {
        uint32_t o[32];
        TA_TMEM_LD32(tbase + 128 + cc * 32, o);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          __half2 hv[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            hv[e] = __floats2half2_rn(__uint_as_float(o[c * 8 + 2 * e]) * f, __uint_as_float(o[c * 8 + 2 * e + 1]) * f);
          const int chunk = cc * 4 + c;
          *reinterpret_cast<uint4*>(stg + lane * (HD * 2) + ((chunk ^ (lane % CH)) << 4)) =
              *reinterpret_cast<uint4*>(hv);
        }
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
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
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

cudaError_t launch_prefill(const turbo_params_t* p, int B, int N, int Nk, int Hq, int Hkv, int causal, const __half* q,
                           const __half* k1, const __half* v1t, const float* k1s, const float* v1s, __half* o,
                           float* lse, cudaStream_t st, const int8_t* q1_in, const float* sq_in) {
  const int HD = p->head_dim, BC = p->block_kv, Tc = (Nk + BC - 1) / BC;
  CUtensorMap tmk, tmv;
  // K [Nk][HD] fp16 codes; boxes of 64 channels x B_c keys (128-B rows, SW128)
  if (!make_map_3d(&tmk, k1, HD, Nk, (uint64_t)B * Hkv, HD * 2, (uint64_t)Nk * HD * 2, 64, BC,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_FLOAT16))
    return cudaErrorInvalidValue;
  // V^T blocks [B_c][HD] of fp16 codes; boxes of 64 keys x HD channels (128-B rows)
  if (!make_map_3d(&tmv, v1t, BC, HD, (uint64_t)B * Hkv * Tc, BC * 2, (uint64_t)HD * BC * 2, 64, HD,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_FLOAT16))
    return cudaErrorInvalidValue;
  PrefillArgs a;
  a.q = q;
  a.q1_in = q1_in;
  a.sq_in = sq_in;
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
  a.scale_fp16 = p->scale_fp16;
  const int G = Hq / Hkv;
  const bool pair = (G % 2) == 0;  // slots = two heads of a GQA group, else two adjacent query tiles
  a.n_qtiles = (N + kTileM - 1) / kTileM;
  {
    static const int sms = [] {  // (thread-safe one-time init; one device per process)
      int dev = 0, n = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
      return n;
    }();
    a.q_prefetch = sms;  // one CTA per SM: the CTA a wave later
    if (const char* e = getenv("TURBO_PREFILL_QPF")) a.q_prefetch = atoi(e) * sms / 4;  // A/B: quarter waves
  }
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
  const bool prow = p->p_scale_rows != 0;
#define TA_LAUNCH_S(HDV, TAPV, TPV, PRV, BCV, SFV)                                                              \
  {                                                                                                            \
    const size_t smem = sizeof(PrefillSmem<HDV, BCV>) + 1024;                                                 \
    cudaFuncSetAttribute(prefill_kernel<HDV, TAPV, TPV, PRV, BCV, SFV>,                                       \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);                              \
    prefill_kernel<HDV, TAPV, TPV, PRV, BCV, SFV><<<grid, 384, smem, st>>>(tmk, tmv, a);                      \
  }
#define TA_LAUNCH_B(HDV, TAPV, TPV, PRV, BCV) \
  if (p->sas_fp16) TA_LAUNCH_S(HDV, TAPV, TPV, PRV, BCV, true) else TA_LAUNCH_S(HDV, TAPV, TPV, PRV, BCV, false)
#define TA_LAUNCH_T(HDV, TAPV, TPV, PRV) \
  if (BC == 64) TA_LAUNCH_B(HDV, TAPV, TPV, PRV, 64) else TA_LAUNCH_B(HDV, TAPV, TPV, PRV, 128)
#define TA_LAUNCH_R(HDV, TAPV, TPV) \
  if (prow) TA_LAUNCH_T(HDV, TAPV, TPV, true) else TA_LAUNCH_T(HDV, TAPV, TPV, false)
#define TA_LAUNCH_P(HDV, TAPV) \
  if (pair) TA_LAUNCH_R(HDV, TAPV, false) else TA_LAUNCH_R(HDV, TAPV, true)
#define TA_LAUNCH(HDV) \
  if (a.has_tap) TA_LAUNCH_P(HDV, true) else TA_LAUNCH_P(HDV, false)
  if (HD == 128) TA_LAUNCH(128) else TA_LAUNCH(64)
#undef TA_LAUNCH
#undef TA_LAUNCH_P
#undef TA_LAUNCH_R
#undef TA_LAUNCH_T
#undef TA_LAUNCH_B
#undef TA_LAUNCH_S
  return cudaGetLastError();
}
}  // namespace ta_host
