// projection.cu -- the Q projection with the stage-1 Q quantisation fused into its epilogue
// (Sec. 5: "we fused the QKV projection with quantization (Eq. 9)"; NEXT-3).
//
//   Q = X W_q^T   X fp16 [T = B N][D], W_q fp16 [Hq d][D] (one row per output feature)
//   -> rounded to fp16, the projection's output precision
//   -> stage 1 per (b, query head, B_r-row block): s_Q = max|Q| / 119, Q^q1 = rne(Q 119 / max|Q|)
//      (Alg. 1; exactly the prefill prologue's arithmetic, R-2 / R-3)
//
// so that turbo_attention_prefill_q1 reads INT8 Q^q1 (d bytes per row) instead of FP16 Q (2d bytes)
// and Q is never written or re-read in FP16.
//
// One CTA per (128-token tile of one sequence, 256 output features = 256 / d heads); 192 threads;
// CL = 2: clusters of two CTAs on consecutive token tiles share the W tile -- each loads one half
// and multicasts it to both (TMA .multicast::cluster), halving the W stream from L2:
//   warp 0      TMA producer: X [128 x 64] and W [256 x 64] fp16 tiles (128B swizzle), 4-stage ring;
//   warp 1      single-thread tcgen05.mma.kind::f16 issuer, M = 128, N = 256, K = 16, fp32 accumulator
//               in 256 TMEM columns (warp 1 also owns TMEM);
//   warps 2-5   epilogue, thread = token row = TMEM lane (warp w reads lane quadrant w % 4): per head the
//               row's d accumulators -> fp16 -> |max| -> the B_r block max across the quadrant warps
//               (shared memory + named barrier) -> codes packed 4 per word, stored row-contiguous.
#include <algorithm>
#include <cstring>

#include "common.cuh"

namespace ta {

constexpr int kPM = 128, kPN = 256, kPK = 64, kPStages = 4;

struct ProjSmem {
  __half a[kPStages][kPM * kPK];  // X tile, K-major, 128-B rows (SW128)
  __half b[kPStages][kPN * kPK];  // W tile, K-major, 128-B rows (SW128)
  uint64_t full[kPStages], empty[kPStages], acc_full[2], acc_empty[2];
  uint32_t tmem_base;
  float red[kPN / 64][4];  // [head][quadrant] row-block maxima
};

struct ProjArgs {
  int8_t* q1;    // [T][Hq][d]
  float* sq;     // [B][Hq][ceil(N / B_r)]
  __half* q16;   // [T][Hq][d] or NULL
  int B, N, D, Hq, HD, block_q, m_tiles, scale_fp16;
};

TA_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
TA_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
TA_DEV void tma_load_2d_mc(void* smem_dst, const void* desc, uint64_t* bar, int c0, int c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(desc), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
TA_DEV void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// Persistent: the grid (a multiple of the cluster size, at most one CTA per SM) walks the tiles --
// (128-token tile, 256-feature tile) pairs of CL consecutive token tiles sharing a feature tile, feature
// tiles outermost -- and keeps two accumulators in TMEM (2 x 256 columns), so the producer and the MMA
// issuer run ahead into the next tile while the epilogue drains the previous one.
template <int HD, int CL>
__global__ void __launch_bounds__(192, 1)
    q_projection_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
                        const __grid_constant__ ProjArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  ProjSmem& sm = *reinterpret_cast<ProjSmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ksteps = args.D / kPK;
  const uint32_t crank = CL > 1 ? cluster_rank() : 0;
  const int mtot = args.m_tiles * args.B;               // token tiles over all sequences
  const int groups = (mtot / CL) * (args.Hq * HD / kPN);  // cluster work units
  const int g0 = blockIdx.x / CL, gstep = gridDim.x / CL;
  auto tile_of = [&](int g, int& b, int& row0, int& n0) {
    const int mx = (g % (mtot / CL)) * CL + (int)crank, ny = g / (mtot / CL);
    b = mx / args.m_tiles;
    row0 = (mx % args.m_tiles) * kPM;
    n0 = ny * kPN;
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], CL);  // one MMA commit per CTA of the cluster (both read the shared W)
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.acc_full[i], 1);
      mbar_init(&sm.acc_empty[i], 4);  // one arrival per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&sm.tmem_base, 2 * kPN);
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync_all();  // the peer's barriers are initialised before any multicast
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch_desc(&tm_x);
      tma_prefetch_desc(&tm_w);
      int kk = 0;  // k-steps issued by this CTA over all its tiles (ring position)
      for (int g = g0; g < groups; g += gstep) {
        int b, row0, n0;
        tile_of(g, b, row0, n0);
        const int xrow = b * args.N + row0;
        for (int k = 0; k < ksteps; ++k, ++kk) {
          const int st = kk % kPStages, n = kk / kPStages;
          if (n > 0) mbar_wait(&sm.empty[st], (n - 1) & 1);
          mbar_expect_tx(&sm.full[st], (kPM + kPN) * kPK * 2);
          tma_load_2d(sm.a[st], &tm_x, &sm.full[st], k * kPK, xrow);
          if (CL == 1) {
            tma_load_2d(sm.b[st], &tm_w, &sm.full[st], k * kPK, n0);
          } else {  // this CTA's half of the W tile, into both CTAs' stage (same offsets)
            constexpr int HALF = kPN / 2;
            tma_load_2d_mc(sm.b[st] + crank * HALF * kPK, &tm_w, &sm.full[st], k * kPK, n0 + (int)crank * HALF,
                           (uint16_t)0x3);
          }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_f16(kPM, kPN);
    int kk = 0, it = 0;
    for (int g = g0; g < groups; g += gstep, ++it) {
      const int ab = it & 1;
      if (it >= 2) mbar_wait(&sm.acc_empty[ab], ((it >> 1) - 1) & 1);  // the epilogue drained this buffer
      tc_fence_after();
      const uint32_t tacc = tmem + ab * kPN;
      for (int k = 0; k < ksteps; ++k, ++kk) {
        const int st = kk % kPStages;
        mbar_wait(&sm.full[st], (kk / kPStages) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t aa = smem_u32(sm.a[st]), ba = smem_u32(sm.b[st]);
#pragma unroll
          for (int ks = 0; ks < kPK / 16; ++ks)
            mma_f16_ss(tacc, smem_desc(aa + ks * 32, 1024, kSw128), smem_desc(ba + ks * 32, 1024, kSw128), idesc,
                       (k | ks) != 0);
          if (CL == 1) mma_commit(&sm.empty[st]);
          else mma_commit_mc(&sm.empty[st], (uint16_t)0x3);  // frees the stage in both CTAs
          if (k == ksteps - 1) mma_commit(&sm.acc_full[ab]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2-5)
    const int qd = warp & 3, r = qd * 32 + lane;
    const int nbq = (args.N + args.block_q - 1) / args.block_q;
    constexpr int NH = kPN / HD;  // heads of a tile
    int it = 0;
    for (int g = g0; g < groups; g += gstep, ++it) {
      int b, row0, n0;
      tile_of(g, b, row0, n0);
      const int ab = it & 1, row = row0 + r;
      const bool row_ok = row < args.N;
      const uint32_t tq = tmem + ((uint32_t)(qd * 32) << 16) + ab * kPN;
      mbar_wait(&sm.acc_full[ab], (it >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int hh = 0; hh < NH; ++hh) {
        const int head = (n0 / HD) + hh;
        // pass 1: the row's |max| over its d fp16 outputs (RNE of the fp32 accumulators)
        float qa = 0.f;
#pragma unroll
        for (int cc = 0; cc < HD / 32; ++cc) {
          uint32_t acc[32];
          TA_TMEM_LD32(tq + hh * HD + cc * 32, acc);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float2 f =
                __half22float2(__floats2half2_rn(__uint_as_float(acc[2 * e]), __uint_as_float(acc[2 * e + 1])));
            qa = fmaxf(qa, fmaxf(fabsf(f.x), fabsf(f.y)));
          }
        }
        if (!row_ok) qa = 0.f;
        qa = warp_max_nonneg(qa);
        if (lane == 0) sm.red[hh][qd] = qa;
        named_bar_sync(1, 128);
        const int half = args.block_q == 64 ? (r >> 6) : 0;
        const float a_q = args.block_q == 64
                              ? fmaxf(sm.red[hh][2 * half], sm.red[hh][2 * half + 1])
                              : fmaxf(fmaxf(sm.red[hh][0], sm.red[hh][1]), fmaxf(sm.red[hh][2], sm.red[hh][3]));
        const float inv_q = a_q > 0.f ? div_119_by(a_q) : 0.f;
        const float s_q = st1_scale(div_by_119(a_q), args.scale_fp16);  // (FP16 variant: R-29)
        const int rb = (row0 + (args.block_q == 64 ? 64 * half : 0)) / args.block_q;  // row block in the sequence
        if ((r & (args.block_q - 1)) == 0 && rb < nbq) args.sq[((size_t)b * args.Hq + head) * nbq + rb] = s_q;
        // pass 2: the same accumulators again -> fp16 -> codes (and the fp16 Q if asked), row-contiguous
        const size_t base = (((size_t)b * args.N + row) * args.Hq + head) * HD;
#pragma unroll
        for (int cc = 0; cc < HD / 32; ++cc) {
          uint32_t acc[32];
          TA_TMEM_LD32(tq + hh * HD + cc * 32, acc);
          tmem_ld_wait();
          uint32_t hq[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const __half2 h2 = __floats2half2_rn(__uint_as_float(acc[2 * e]), __uint_as_float(acc[2 * e + 1]));
            hq[e] = *reinterpret_cast<const uint32_t*>(&h2);
          }
          if (row_ok) {
            uint4* dst = reinterpret_cast<uint4*>(args.q1 + base + cc * 32);
#pragma unroll
            for (int c16 = 0; c16 < 2; ++c16) {
              uint32_t w[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&hq[c16 * 8 + 2 * e]));
                const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&hq[c16 * 8 + 2 * e + 1]));
                w[e] = pack4_lo(rint_prod_bits(f0.x, inv_q), rint_prod_bits(f0.y, inv_q),
                                rint_prod_bits(f1.x, inv_q), rint_prod_bits(f1.y, inv_q));
              }
              dst[c16] = make_uint4(w[0], w[1], w[2], w[3]);
            }
            if (args.q16) {
              uint4* d16 = reinterpret_cast<uint4*>(args.q16 + base + cc * 32);
#pragma unroll
              for (int c8 = 0; c8 < 4; ++c8)
                d16[c8] = make_uint4(hq[4 * c8], hq[4 * c8 + 1], hq[4 * c8 + 2], hq[4 * c8 + 3]);
            }
          }
        }
        if (hh == NH - 1) {  // every TMEM read of this buffer is done: hand it back to the MMA issuer
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.acc_empty[ab]);
        }
        named_bar_sync(1, 128);  // sm.red is rewritten by the next head
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync_all();  // no CTA leaves while its peer may still multicast into it
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 2 * kPN);
  }
}

}  // namespace ta

// ---------------------------------------------------------------------------
namespace ta_host {
using namespace ta;

typedef CUresult (*EncodeTiled2Fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static bool make_map_2d_f16(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint32_t box_cols,
                            uint32_t box_rows) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
    return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return reinterpret_cast<EncodeTiled2Fn>(fn)(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims,
                                              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_q_projection(const turbo_params_t* p, int B, int N, int D, int Hq, const __half* x, const __half* wq,
                                int8_t* q1, float* sq, __half* q16, cudaStream_t st) {
  const int HD = p->head_dim;
  CUtensorMap tmx, tmw;
  if (!make_map_2d_f16(&tmx, x, D, (uint64_t)B * N, kPK, kPM)) return cudaErrorInvalidValue;
  const bool pair = ((N + kPM - 1) / kPM * B) % 2 == 0;  // clusters of two token tiles sharing the W tile
  // W boxes: the whole 256-feature tile, or (pair) the half each CTA of the cluster multicasts
  if (!make_map_2d_f16(&tmw, wq, D, (uint64_t)Hq * HD, kPK, pair ? kPN / 2 : kPN)) return cudaErrorInvalidValue;
  ProjArgs a;
  a.q1 = q1;
  a.sq = sq;
  a.q16 = q16;
  a.B = B;
  a.N = N;
  a.D = D;
  a.Hq = Hq;
  a.HD = HD;
  a.block_q = p->block_q;
  a.m_tiles = (N + kPM - 1) / kPM;
  a.scale_fp16 = p->scale_fp16;
  const size_t smem = sizeof(ProjSmem) + 1024;
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int cl = pair ? 2 : 1;
  const int groups = (a.m_tiles * B / cl) * (Hq * HD / kPN);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(std::max(1, sms / cl) * cl));
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = pair ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // persistent grid: as many clusters as can be resident at once (never a second wave), at most the tiles
#define TA_PROJ(HDV, CLV)                                                                                  \
  {                                                                                                        \
    cudaFuncSetAttribute(q_projection_kernel<HDV, CLV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    int ncl = 0;                                                                                           \
    if (cudaOccupancyMaxActiveClusters(&ncl, q_projection_kernel<HDV, CLV>, &cfg) != cudaSuccess || ncl < 1) \
      ncl = std::max(1, sms / CLV);                                                                        \
    cfg.gridDim = dim3((unsigned)(std::min(groups, ncl) * CLV));                                           \
    cudaError_t e = cudaLaunchKernelEx(&cfg, q_projection_kernel<HDV, CLV>, tmx, tmw, a);                  \
    return e != cudaSuccess ? e : cudaGetLastError();                                                      \
  }
  if (HD == 128) {
    if (pair) TA_PROJ(128, 2) else TA_PROJ(128, 1)
  } else {
    if (pair) TA_PROJ(64, 2) else TA_PROJ(64, 1)
  }
#undef TA_PROJ
}
}  // namespace ta_host
