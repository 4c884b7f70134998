// Issue/pipe throughput of FFMA, FFMA2, FADD2.RM, FMUL2, I2FP, FSEL, FMNMX3 and
// SHFL.IDX per SM sub-partition: W warps per CTA, one CTA per SM, 8 independent
// chains per thread.  Prints warp-instructions per clock per SMSP.
#include <cstdio>
#include "common.cuh"

using namespace ta;

template <int OP>
__global__ void __launch_bounds__(1024, 1) kern(int iters, float seed, unsigned long long* cyc, float* sink) {
  float a[8];
  f32x2 p[8];
  int ii[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    a[k] = seed + k + threadIdx.x;
    p[k] = pk2(a[k], a[k] + 1.f);
    ii[k] = threadIdx.x + k;
  }
  const f32x2 c2 = pk2(1.0001f, 0.9999f), d2 = pk2(1e-7f, 2e-7f);
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) a[k] = __fmaf_rn(a[k], 1.0001f, 1e-7f);
      if (OP == 1) p[k] = fma2(p[k], c2, d2);
      if (OP == 2) p[k] = add2_rd(p[k], d2);
      if (OP == 3) p[k] = mul2(p[k], c2);
      if (OP == 4) a[k] = __int2float_rn(ii[k] + __float_as_int(a[k]));
      if (OP == 5) a[k] = a[k] > 0.5f ? a[k] * 1.0001f : a[k];  // FSETP + FSEL(ish)
      if (OP == 6) a[k] = fmaxf(a[k], fmaxf(a[(k + 1) & 7], seed));
      if (OP == 7) a[k] = __uint_as_float(__shfl_sync(0xffffffffu, __float_as_uint(a[k]), ii[k] & 31));
      if (OP == 8) ii[k] = ii[k] * 3 + 1;
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k] + lo2(p[k]) + hi2(p[k]) + ii[k];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
void run(const char* name, int warps) {
  unsigned long long* cyc;
  float* sink;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&sink, 148 * 1024 * 4);
  const int iters = 4096;
  kern<OP><<<148, 32 * warps>>>(16, 1.f, cyc, sink);
  cudaMemset(cyc, 0, 8);
  kern<OP><<<148, 32 * warps>>>(iters, 1.f, cyc, sink);
  unsigned long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double clk = (double)h / 148;
  const double winst = (double)iters * 8 * warps;  // per SM
  printf("%-10s warps %2d: %.3f warp-inst/clk/SMSP\n", name, warps, winst / clk / 4);
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  for (int w : {8, 16, 32}) {
    run<0>("FFMA", w);
    run<1>("FFMA2", w);
    run<2>("FADD2.RM", w);
    run<3>("FMUL2", w);
    run<4>("IADD+I2F", w);
    run<5>("FSETP/SEL", w);
    run<6>("FMNMX", w);
    run<7>("SHFL.IDX", w);
    run<8>("IMAD", w);
  }
  return 0;
}
