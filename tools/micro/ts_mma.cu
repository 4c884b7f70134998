// Layout probe for the TMEM-A form of tcgen05.mma kind::f16 (D[tmem] += A[tmem] . B[smem]):
// 128 threads write A [128 x 64] fp16 into TMEM with tcgen05.st.32x32b.x32 (thread = row =
// lane, column c = the fp16 pair (2c, 2c+1)), B = V^T [N][64] fp16 in smem as 128-B
// SW128 rows (the prefill's V tile layout), 4 MMAs of K = 16 (A address + 8 columns
// each).  Checks D against a host GEMM for both orders of the halves inside a column.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_2412_08585_b200/csrc
//        -I ../../include ts_mma.cu -o ts_mma -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

using namespace ta;
constexpr int N = 128;

__global__ void __launch_bounds__(128, 1) ts_kernel(const __half* a, const __half* b, float* d, int iters,
                                                     unsigned long long* cyc) {
  __shared__ __align__(1024) __half bs[N * 64];
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5;
  // B rows (n) of 64 halves = 128 B, SW128: 16-B chunk c of row n at chunk c ^ (n & 7)
  for (int i = t; i < N * 8; i += 128) {
    const int n = i >> 3, c = i & 7;
    *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(bs) + n * 128 + ((c ^ (n & 7)) << 4)) =
        *reinterpret_cast<const uint4*>(b + n * 64 + c * 8);
  }
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 256);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  {
    uint32_t r[32];
    for (int c = 0; c < 32; ++c) {
      __half2 h2 = __halves2half2(a[t * 64 + 2 * c], a[t * 64 + 2 * c + 1]);
      r[c] = *reinterpret_cast<uint32_t*>(&h2);
    }
    TA_TMEM_ST32(tm + ((uint32_t)(warp * 32) << 16), r);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  long long c0 = clock64();
  if (t == 0) {
    constexpr uint32_t idesc = idesc_f16(128, N);
    const uint32_t ba = smem_u32(bs);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm + 128),
            "r"(tm + ks * 8), "l"(smem_desc(ba + ks * 32, 1024, kSw128)), "r"(idesc), "r"((it | ks) ? 1 : 0)
            : "memory");
      }
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  long long c1 = clock64();
  if (t == 0) *cyc = (unsigned long long)(c1 - c0);
  tc_fence_after();
  {
    uint32_t r[32];
    for (int cc = 0; cc < N / 32; ++cc) {
      TA_TMEM_LD32(tm + ((uint32_t)(warp * 32) << 16) + 128 + cc * 32, r);
      tmem_ld_wait();
      for (int e = 0; e < 32; ++e) d[t * N + cc * 32 + e] = __uint_as_float(r[e]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tm, 256);
  }
}

int main() {
  std::vector<__half> ha(128 * 64), hb(N * 64);
  std::vector<float> fa(128 * 64), fb(N * 64);
  srand(1);
  for (int i = 0; i < 128 * 64; ++i) fa[i] = (float)(rand() % 239 - 119) / 64.0f, ha[i] = __float2half(fa[i]);
  for (int i = 0; i < N * 64; ++i) fb[i] = (float)(rand() % 239 - 119), hb[i] = __float2half(fb[i]);
  __half *da, *db;
  float* dd;
  unsigned long long* cyc;
  cudaMalloc(&da, ha.size() * 2);
  cudaMalloc(&db, hb.size() * 2);
  cudaMalloc(&dd, 128 * N * 4);
  cudaMalloc(&cyc, 8);
  cudaMemcpy(da, ha.data(), ha.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice);
  ts_kernel<<<1, 128>>>(da, db, dd, 1, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("ts_mma: CUDA error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> hd(128 * N);
  cudaMemcpy(hd.data(), dd, hd.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0, bad_sw = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0, ref_sw = 0;
      for (int k = 0; k < 64; ++k) {
        ref += (double)fa[m * 64 + k] * fb[n * 64 + k];
        ref_sw += (double)fa[m * 64 + (k ^ 1)] * fb[n * 64 + k];
      }
      if (hd[m * N + n] != (float)ref) ++bad;
      if (hd[m * N + n] != (float)ref_sw) ++bad_sw;
    }
  printf("ts_mma kind::f16 A-from-TMEM: mismatches %d (low half = even k), %d (swapped halves); D[0][0]=%g\n", bad,
         bad_sw, hd[0]);
  const int iters = 4096;
  ts_kernel<<<148, 128>>>(da, db, dd, iters, cyc);
  cudaDeviceSynchronize();
  unsigned long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("ts_mma 128x%dx64 per CTA: %.1f clk per MMA group (4 x K16) -> %.0f fp16 MAC/clk/SM\n", N,
         (double)c / iters, 128.0 * N * 64 * iters / c);
  return bad == 0 ? 0 : 2;
}
