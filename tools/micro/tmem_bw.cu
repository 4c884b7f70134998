// TMEM -> register bandwidth microbenchmark (tcgen05.ld.32x32b.x32 + wait::ld).
// One CTA per SM, W warps (W/4 per TMEM lane quadrant), each warp repeatedly
// loads 32 columns x 32 lanes x 4 B = 4 KB from its quadrant.  Prints bytes per
// SM clock.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_2412_08585_b200/csrc tmem_bw.cu
#include <cstdio>
#include "common.cuh"

template <int W, int X>
__global__ void __launch_bounds__(32 * W, 1) tmem_bw(int iters, unsigned long long* cyc, unsigned* sink) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ta::tmem_alloc(&tbase, 512);
  ta::tc_fence_before();
  __syncthreads();
  ta::tc_fence_after();
  const uint32_t t = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + 64 * (warp >> 2);
  uint32_t acc = 0;
  __syncthreads();
  const long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t r[32];
#pragma unroll
    for (int x = 0; x < X; ++x) {
      TA_TMEM_LD32(t + 32 * x, r);
      if (x == X - 1) ta::tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 32; ++e) acc += r[e];
    }
  }
  __syncthreads();
  const long long c1 = clock64();
  if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(c1 - c0));
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  ta::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ta::tc_fence_after();
    ta::tmem_dealloc(tbase, 512);
  }
}

template <int W, int X>
void run(int sms) {
  unsigned long long* cyc;
  unsigned* sink;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&sink, sms * 32 * W * 4);
  const int iters = 2000;
  tmem_bw<W, X><<<sms, 32 * W>>>(10, cyc, sink);
  cudaMemset(cyc, 0, 8);
  tmem_bw<W, X><<<sms, 32 * W>>>(iters, cyc, sink);
  unsigned long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double per_cta = (double)h / sms;
  const double bytes = (double)iters * X * W * 4096.0;
  printf("warps %2d  ld.x32 per wait %d : %.1f B/clk/SM  (%.0f clk per x32 ld per warp)\n", W, X, bytes / per_cta,
         per_cta / (iters * X));
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  int sms = 148;
  run<4, 1>(sms);
  run<4, 2>(sms);
  run<4, 4>(sms);
  run<8, 1>(sms);
  run<8, 2>(sms);
  run<8, 4>(sms);
  run<16, 2>(sms);
  return 0;
}
