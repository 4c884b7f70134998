// prefill.cu -- Algorithm 1 (TurboAttention prefill) on sm_100a.
//
// One CTA = one (batch, query head, 128-row query tile); the tile holds two
// B_r = 64 quantisation blocks (or one B_r = 128 block).  Warp roles:
//   warp 0      TMA producer: K_j [64 x d] and V_j^T [d x 64] INT8 tiles into a
//               3-stage smem ring (cp.async.bulk.tensor, 128B/64B swizzle).
//   warp 1      TMEM owner + single-thread tcgen05.mma issuer (kind::i8):
//               S_j = Q^q1 K_j^q1^T -> TMEM (int32, double-buffered) and
//               PV_j = Q(P~_j) V_j^q1 -> TMEM (int32).
//   warps 4-7   softmax/correction warpgroup, thread = query row = TMEM lane:
//               Q stage-1 quantisation, integer row max, SAS (LUT x POLY) in
//               registers, P tile scale + INT8 codes -> smem (A operand of the
//               PV MMA), and O = alpha O + s_P s_V PV_int in FP32 registers
//               one tile behind (overlapping the next MMA).
#include <climits>
#include <cstring>

#include "common.cuh"

namespace ta {

constexpr int kStages = 3;
constexpr int kTileM = 128;
constexpr int kTmemCols = 256;  // S0 [0,64) S1 [64,128) PV [128, 128 + d)

template <int HD>
struct PrefillSmem {
  int8_t q1[kTileM * HD];         // Q^q1, K-major, swizzled rows of HD bytes
  int8_t k[kStages][kBc * HD];    // K_j^q1 [64][HD]
  int8_t v[kStages][HD * kBc];    // V_j^q1 transposed [HD][64]
  int8_t p[2][kTileM * kBc];      // Q(P~) [128][64], SW64
  uint64_t kv_full[kStages], kv_empty[kStages], s_full[2], s_free[2], p_full[2], pv_full, pv_free, q_ready;
  uint32_t tmem_base;
  float red_a[4];
  float red_p[2][4];
};

struct PrefillArgs {
  const __half* q;
  __half* o;
  float* lse;
  const float* k1s;
  const float* v1s;
  int B, N, Hq, Hkv, causal, block_q, alpha_mode, n_qtiles;
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
TA_DEV uint32_t p_swz(int r, int chunk) { return r * 64 + ((chunk ^ ((r >> 1) & 3)) << 4); }

template <int HD>
__global__ void __launch_bounds__(256, 1)
    prefill_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                   const __grid_constant__ PrefillArgs args) {
  extern __shared__ uint8_t smem_raw[];
  PrefillSmem<HD>& sm =
      *reinterpret_cast<PrefillSmem<HD>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // Heaviest (last) query tiles first for causal load balance.
  const int BH = args.B * args.Hq;
  const int it = args.n_qtiles - 1 - (int)(blockIdx.x / BH);
  const int bh = blockIdx.x % BH, b = bh / args.Hq, h = bh % args.Hq;
  const int kvh = h / (args.Hq / args.Hkv);
  const int N = args.N, Tc = (N + kBc - 1) / kBc;
  const int last_row = min(it * kTileM + kTileM - 1, N - 1);
  const int nkv = args.causal ? min(Tc, last_row / kBc + 1) : Tc;
  const size_t bkv = (size_t)b * args.Hkv + kvh;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.kv_full[s], 1);
      mbar_init(&sm.kv_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.s_full[s], 1);
      mbar_init(&sm.s_free[s], 128);
      mbar_init(&sm.p_full[s], 128);
    }
    mbar_init(&sm.pv_full, 1);
    mbar_init(&sm.pv_free, 128);
    mbar_init(&sm.q_ready, 128);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&sm.tmem_base, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      for (int j = 0; j < nkv; ++j) {
        const int st = j % kStages, n = j / kStages;
        if (n > 0) mbar_wait(&sm.kv_empty[st], (n - 1) & 1);
        mbar_expect_tx(&sm.kv_full[st], 2 * kBc * HD);
        tma_load_3d(sm.k[st], &tm_k, &sm.kv_full[st], 0, j * kBc, (int)bkv);
        tma_load_3d(sm.v[st], &tm_v, &sm.kv_full[st], 0, 0, (int)(bkv * Tc + j));
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t kLayQK = HD == 128 ? kSw128 : kSw64;
    constexpr uint32_t idesc_qk = idesc_i8(kTileM, kBc, true, true);
    constexpr uint32_t idesc_pv = idesc_i8(kTileM, HD, false, true);
    const uint32_t q1a = smem_u32(sm.q1);
    mbar_wait(&sm.q_ready, 0);
    tc_fence_after();
    for (int j = 0; j <= nkv; ++j) {
      if (j < nkv) {
        const int st = j % kStages, sb = j & 1;
        mbar_wait(&sm.kv_full[st], (j / kStages) & 1);
        if (j >= 2) mbar_wait(&sm.s_free[sb], ((j >> 1) - 1) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t ka = smem_u32(sm.k[st]);
#pragma unroll
          for (int ks = 0; ks < HD / 32; ++ks)
            mma_i8_ss(tmem + sb * kBc, smem_desc(q1a + ks * 32, 8 * HD, kLayQK), smem_desc(ka + ks * 32, 8 * HD, kLayQK),
                      idesc_qk, ks > 0);
          mma_commit(&sm.s_full[sb]);
        }
        __syncwarp();
      }
      if (j >= 1) {
        const int jj = j - 1, pb = jj & 1, st = jj % kStages;
        mbar_wait(&sm.p_full[pb], (jj >> 1) & 1);
        if (jj >= 1) mbar_wait(&sm.pv_free, (jj - 1) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t pa = smem_u32(sm.p[pb]), va = smem_u32(sm.v[st]);
#pragma unroll
          for (int ks = 0; ks < kBc / 32; ++ks)
            mma_i8_ss(tmem + 2 * kBc, smem_desc(pa + ks * 32, 512, kSw64), smem_desc(va + ks * 32, 512, kSw64),
                      idesc_pv, ks > 0);
          mma_commit(&sm.pv_full);
          mma_commit(&sm.kv_empty[st]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax / correction
    const int qd = warp & 3, r = qd * 32 + lane, row = it * kTileM + r;
    const bool row_ok = row < N;
    const int half = args.block_q == 64 ? (r >> 6) : 0;
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    const float lut_lane = args.sas.lut[lane];
    const float nr_abs = args.sas.nr_abs;
    const bool tap_cta = args.has_tap && args.tap.batch == b && args.tap.head == h &&
                         (args.tap.i_block >> 1) == it;
    const bool tap_row = tap_cta && (args.tap.i_block & 1) == (r >> 6);

    // Q stage-1 quantisation (Alg. 1; per B_r x d block).
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
    qa = warp_max(qa);
    if (lane == 0) sm.red_a[qd] = qa;
    named_bar_sync(1, 128);
    float a_q = args.block_q == 64 ? fmaxf(sm.red_a[2 * half], sm.red_a[2 * half + 1])
                                   : fmaxf(fmaxf(sm.red_a[0], sm.red_a[1]), fmaxf(sm.red_a[2], sm.red_a[3]));
    const float inv_q = a_q > 0.f ? __fdiv_rn(kDiv, a_q) : 0.f;
    const float s_q = __fdiv_rn(a_q, kDiv);
#pragma unroll
    for (int c = 0; c < HD / 16; ++c) {
      uint32_t w[4];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const __half2* hp = reinterpret_cast<const __half2*>(&qraw[2 * c + hh]);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          float2 f0 = __half22float2(hp[2 * e]), f1 = __half22float2(hp[2 * e + 1]);
          w[hh * 2 + e] = (uint32_t)(rint_prod(f0.x, inv_q) & 0xFF) | ((uint32_t)(rint_prod(f0.y, inv_q) & 0xFF) << 8) |
                          ((uint32_t)(rint_prod(f1.x, inv_q) & 0xFF) << 16) |
                          ((uint32_t)(rint_prod(f1.y, inv_q) & 0xFF) << 24);
        }
      }
      *reinterpret_cast<uint4*>(sm.q1 + q1_swz<HD>(r, c)) = make_uint4(w[0], w[1], w[2], w[3]);
      if (tap_row) *reinterpret_cast<uint4*>(args.tap.q1 + (r & 63) * HD + c * 16) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    if (tap_row && (r & 63) == 0) args.tap.s_q[0] = s_q;
    fence_proxy_async();
    mbar_arrive(&sm.q_ready);

    float O[HD];
#pragma unroll
    for (int c = 0; c < HD; ++c) O[c] = 0.f;
    float m = -INFINITY, l = 0.f;
    float alpha_p = 0.f, cpv_p = 0.f;
    bool active_p = false, tap_p = false;
    const int kmax = row_ok ? (args.causal ? row : N - 1) : -1;  // last visible key of this row

    for (int j = 0; j <= nkv; ++j) {
      bool active = false;
      float alpha = 0.f, cpv = 0.f;
      const bool tap_j = tap_row && args.tap.j_block == j;
      if (j < nkv) {
        const int sb = j & 1;
        uint32_t sv[kBc];
        mbar_wait(&sm.s_full[sb], (j >> 1) & 1);
        tc_fence_after();
        TA_TMEM_LD32(tmem + lane_base + sb * kBc, sv);
        TA_TMEM_LD32(tmem + lane_base + sb * kBc + 32, (sv + 32));
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&sm.s_free[sb]);

        const int nvalid = max(0, min(kBc, kmax - j * kBc + 1));
        active = nvalid > 0;
        int smax = INT_MIN;
#pragma unroll
        for (int c = 0; c < kBc; ++c)
          if (c < nvalid) smax = max(smax, (int)sv[c]);
        // S = s_Q s_K Q^q1 K^q1^T scaled by 1/sqrt(d) (R-18)
        const float cqk = __fmul_rn(__fmul_rn(s_q, args.k1s[bkv * Tc + j]), args.scale);
        float m_new = m;
        if (active) {
          m_new = fmaxf(m, __fmul_rn((float)smax, cqk));
          if (m == -INFINITY) alpha = 0.f;
          else if (args.alpha_mode == 1 && m_new == m) alpha = 1.f;
          else alpha = sas_eval_scalar(__fsub_rn(m_new, m), args.sas);
        }
        if (tap_j) {
          for (int c = 0; c < kBc; ++c) args.tap.s_int[(r & 63) * kBc + c] = c < nvalid ? (int)sv[c] : 0;
        }
        // P~ = SAS(S - m_new), masked keys -> 0
        float rsum = 0.f, pmax = 0.f;
#pragma unroll
        for (int c = 0; c < kBc; ++c) {
          const float x = __fmul_rn((float)(int)sv[c], cqk);
          float pt = sas_eval(__fsub_rn(m_new, x), lut_lane, nr_abs);
          pt = c < nvalid ? pt : 0.f;
          rsum += pt;
          pmax = fmaxf(pmax, pt);
          sv[c] = __float_as_uint(pt);
        }
        if (active) {
          l = alpha * l + rsum;  // l = SAS(m_prev - m_new) l + rowsum(P~)
          m = m_new;
        }
        // P scale over the B_r x B_c tile
        pmax = warp_max(pmax);
        if (lane == 0) sm.red_p[sb][qd] = pmax;
        named_bar_sync(1, 128);
        const float a_p = args.block_q == 64
                              ? fmaxf(sm.red_p[sb][2 * half], sm.red_p[sb][2 * half + 1])
                              : fmaxf(fmaxf(sm.red_p[sb][0], sm.red_p[sb][1]), fmaxf(sm.red_p[sb][2], sm.red_p[sb][3]));
        const float inv_p = a_p > 0.f ? __fdiv_rn(kDiv, a_p) : 0.f;
        const float s_p = __fdiv_rn(a_p, kDiv);
        cpv = __fmul_rn(s_p, args.v1s[bkv * Tc + j]);
        // Q(P~) codes in [0, 119] -> smem (A operand of the PV MMA)
        uint8_t* prow = reinterpret_cast<uint8_t*>(sm.p[sb]);
#pragma unroll
        for (int c = 0; c < kBc / 16; ++c) {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int c0 = c * 16 + e * 4;
            w[e] = (uint32_t)rint_prod(__uint_as_float(sv[c0]), inv_p) |
                   ((uint32_t)rint_prod(__uint_as_float(sv[c0 + 1]), inv_p) << 8) |
                   ((uint32_t)rint_prod(__uint_as_float(sv[c0 + 2]), inv_p) << 16) |
                   ((uint32_t)rint_prod(__uint_as_float(sv[c0 + 3]), inv_p) << 24);
          }
          *reinterpret_cast<uint4*>(prow + p_swz(r, c)) = make_uint4(w[0], w[1], w[2], w[3]);
          if (tap_j) *reinterpret_cast<uint4*>(args.tap.p_codes + (r & 63) * kBc + c * 16) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        if (tap_j) {
          args.tap.m_new[r & 63] = m;
          if ((r & 63) == 0) args.tap.s_p[0] = s_p;
        }
        fence_proxy_async();
        mbar_arrive(&sm.p_full[sb]);
      }
      // O = alpha O + s_P s_V Q(P~) V^q1 for the previous tile
      if (j >= 1) {
        mbar_wait(&sm.pv_full, (j - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int cc = 0; cc < HD / 32; ++cc) {
          uint32_t pv[32];
          TA_TMEM_LD32(tmem + lane_base + 2 * kBc + cc * 32, pv);
          tmem_ld_wait();
          if (active_p) {
#pragma unroll
            for (int e = 0; e < 32; ++e) O[cc * 32 + e] = __fmaf_rn(alpha_p, O[cc * 32 + e], cpv_p * (float)(int)pv[e]);
          }
          if (tap_p) {
            for (int e = 0; e < 32; ++e) args.tap.pv_int[(r & 63) * HD + cc * 32 + e] = (int)pv[e];
          }
        }
        tc_fence_before();
        if (j < nkv) mbar_arrive(&sm.pv_free);
      }
      alpha_p = alpha;
      cpv_p = cpv;
      active_p = active;
      tap_p = tap_j;
    }
    // Epilogue: O_i = diag(l)^-1 O, L_i = m + log l
    if (row_ok) {
      const float inv_l = 1.f / l;
      __half* orow = args.o + (((size_t)b * N + row) * args.Hq + h) * HD;
#pragma unroll
      for (int c = 0; c < HD / 8; ++c) {
        __half2 hv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) hv[e] = __floats2half2_rn(O[c * 8 + 2 * e] * inv_l, O[c * 8 + 2 * e + 1] * inv_l);
        reinterpret_cast<uint4*>(orow)[c] = *reinterpret_cast<uint4*>(hv);
      }
      args.lse[((size_t)b * args.Hq + h) * N + row] = m + logf(l);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
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
                        uint64_t s2, uint32_t b0, uint32_t b1, CUtensorMapSwizzle swz) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1, s2};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_prefill(const turbo_params_t* p, int B, int N, int Hq, int Hkv, int causal, const __half* q,
                           const int8_t* k1, const int8_t* v1t, const float* k1s, const float* v1s, __half* o,
                           float* lse, cudaStream_t st) {
  const int HD = p->head_dim, Tc = (N + kBc - 1) / kBc;
  CUtensorMap tmk, tmv;
  const CUtensorMapSwizzle swk = HD == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  if (!make_map_3d(&tmk, k1, HD, N, (uint64_t)B * Hkv, HD, (uint64_t)N * HD, HD, kBc, swk))
    return cudaErrorInvalidValue;
  if (!make_map_3d(&tmv, v1t, kBc, HD, (uint64_t)B * Hkv * Tc, kBc, (uint64_t)HD * kBc, kBc, HD,
                   CU_TENSOR_MAP_SWIZZLE_64B))
    return cudaErrorInvalidValue;
  PrefillArgs a;
  a.q = q;
  a.o = o;
  a.lse = lse;
  a.k1s = k1s;
  a.v1s = v1s;
  a.B = B;
  a.N = N;
  a.Hq = Hq;
  a.Hkv = Hkv;
  a.causal = causal;
  a.block_q = p->block_q;
  a.alpha_mode = p->alpha_mode;
  a.n_qtiles = (N + kTileM - 1) / kTileM;
  a.scale = p->softmax_scale;
  fill_sas_const(&a.sas, p->sas_nr);
  a.has_tap = p->debug_tap != nullptr;
  if (a.has_tap) a.tap = *reinterpret_cast<const turbo_debug_tap_t*>(p->debug_tap);
  else memset(&a.tap, 0, sizeof(a.tap));
  const dim3 grid((unsigned)(a.n_qtiles * B * Hq));
  if (HD == 128) {
    const size_t smem = sizeof(PrefillSmem<128>) + 1024;
    cudaFuncSetAttribute(prefill_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    prefill_kernel<128><<<grid, 256, smem, st>>>(tmk, tmv, a);
  } else {
    const size_t smem = sizeof(PrefillSmem<64>) + 1024;
    cudaFuncSetAttribute(prefill_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    prefill_kernel<64><<<grid, 256, smem, st>>>(tmk, tmv, a);
  }
  return cudaGetLastError();
}
}  // namespace ta_host
