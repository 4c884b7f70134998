// Issue/pipe throughput of the softmax-path instructions not covered by pipe_tp.cu:
// HFMA2, HMUL2, F2FP (cvt.rn.f16x2.f32), PRMT, LOP3, IMNMX, I2F alone, FSEL alone,
// cvt.f32.f16, and two mixes (FFMA2 + LOP3, FFMA2 + I2F) that show which pipes
// co-issue.  W warps per CTA, one CTA per SM, 8 independent chains per thread.
// Prints warp-instructions per clock per SM sub-partition.
#include <cstdio>
#include "common.cuh"

using namespace ta;

template <int OP>
__global__ void __launch_bounds__(1024, 1) kern(int iters, float seed, unsigned long long* cyc, float* sink) {
  float a[8];
  f32x2 p[8];
  uint32_t u[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    a[k] = seed + k + threadIdx.x;
    p[k] = pk2(a[k], a[k] + 1.f);
    u[k] = threadIdx.x * 7 + k;
  }
  const uint32_t h2c = 0x3c003c01u, h2d = 0x00010002u;
  const f32x2 c2 = pk2(1.0001f, 0.9999f), d2 = pk2(1e-7f, 2e-7f);
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(u[k]) : "r"(h2c), "r"(h2d));
      if (OP == 1) asm volatile("mul.rn.f16x2 %0, %0, %1;" : "+r"(u[k]) : "r"(h2c));
      if (OP == 2) {
        uint32_t r;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[k]), "f"(a[(k + 1) & 7]));
        a[k] = __uint_as_float(r);
      }
      if (OP == 3) u[k] = __byte_perm(u[k], u[(k + 1) & 7], 0x5410);
      if (OP == 4) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[k]) : "r"(u[(k + 1) & 7]), "r"(h2c));
      if (OP == 5) asm volatile("max.s32 %0, %0, %1;" : "+r"(u[k]) : "r"(u[(k + 3) & 7]));
      if (OP == 6) asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(a[k]) : "r"(u[k] ^ __float_as_uint(a[k])));
      if (OP == 7) {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.gt.f32 q, %1, 0f3F000000;\n\tselp.f32 %0, %1, %2, q;\n\t}"
                     : "=f"(a[k])
                     : "f"(a[k]), "f"(seed));
      }
      if (OP == 8) {
        float f;
        asm volatile("{\n\t.reg .b16 h;\n\tmov.b32 {h, _}, %1;\n\tcvt.f32.f16 %0, h;\n\t}" : "=f"(f) : "r"(u[k]));
        u[k] = __float_as_uint(f) + 1;
      }
      if (OP == 9) {
        p[k] = fma2(p[k], c2, d2);
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[k]) : "r"(u[(k + 1) & 7]), "r"(h2c));
      }
      if (OP == 10) {
        p[k] = fma2(p[k], c2, d2);
        asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(a[k]) : "r"(u[k] ^ __float_as_uint(a[k])));
      }
      if (OP == 11) {
        p[k] = fma2(p[k], c2, d2);
        asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(u[k]) : "r"(h2c), "r"(h2d));
      }
      if (OP == 12) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[k]) : "f"(a[(k + 1) & 7]), "f"(seed));
      if (OP == 14) p[k] = fma2(p[k], pk2(1.0001f, 1.0001f), pk2(1e-7f, 1e-7f));  // FFMA2 imm b, c
      if (OP == 15) p[k] = fma2(p[k], p[(k + 1) & 7], p[(k + 2) & 7]);           // FFMA2 3-reg
      if (OP == 16) p[k] = add2(p[k], pk2(1e-7f, 1e-7f));                       // FADD2 imm
      if (OP == 17) p[k] = add2(p[k], p[(k + 1) & 7]);                          // FADD2 reg pair
      if (OP == 18) p[k] = mul2(p[k], pk2(seed, seed));                          // FMUL2 scalar-reg broadcast
      if (OP == 19) a[k] = fmaf(a[k], 1.0001f, 1e-7f);                           // FFMA imm
      if (OP == 20) a[k] = fmaf(a[k], a[(k + 1) & 7], a[(k + 2) & 7]);           // FFMA 3-reg
      if (OP == 21) p[k] = fma2(p[k], pk2(seed, seed), pk2(1e-7f, 1e-7f));       // FFMA2 scalar b, imm c
      if (OP == 22) asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(a[k]) : "r"(u[k]));  // I2F alone (no dep)
      if (OP == 23) {                                                          // FADD2 imm + I2F
        p[k] = add2(p[k], pk2(1e-7f, 1e-7f));
        asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(a[k]) : "r"(u[k] ^ k));
      }
      if (OP == 24) {  // REDUX max
        u[k] = __reduce_max_sync(0xffffffffu, u[k] + k);
      }
      if (OP == 13) {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.gt.f32 q, %1, 0f3F000000;\n\tselp.f32 %0, %1, %2, q;\n\t}"
                     : "=f"(a[k])
                     : "f"(a[k]), "f"(seed));
        p[k] = fma2(p[k], c2, d2);
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k] + lo2(p[k]) + hi2(p[k]) + (float)u[k];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
void run(const char* name, int warps, int per) {
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
  const double winst = (double)iters * 8 * warps * per;  // per SM
  printf("%-14s warps %2d: %.3f warp-inst/clk/SMSP\n", name, warps, winst / clk / 4);
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  for (int w : {8, 16}) {
    run<0>("HFMA2", w, 1);
    run<1>("HMUL2", w, 1);
    run<2>("F2FP.F16x2", w, 1);
    run<3>("PRMT", w, 1);
    run<4>("LOP3", w, 1);
    run<5>("IMNMX", w, 1);
    run<6>("I2F(+LOP)", w, 2);
    run<7>("FSETP+SEL", w, 2);
    run<8>("F16->F32(+IADD)", w, 2);
    run<9>("FFMA2+LOP3", w, 2);
    run<10>("FFMA2+I2F+LOP", w, 3);
    run<11>("FFMA2+HFMA2", w, 2);
    run<12>("FMNMX3", w, 1);
    run<13>("FSETP+SEL+FFMA2", w, 3);
    run<14>("FFMA2 imm", w, 1);
    run<15>("FFMA2 3reg", w, 1);
    run<16>("FADD2 imm", w, 1);
    run<17>("FADD2 reg", w, 1);
    run<18>("FMUL2 bcast", w, 1);
    run<19>("FFMA imm", w, 1);
    run<20>("FFMA 3reg", w, 1);
    run<21>("FFMA2 bc+imm", w, 1);
    run<22>("I2F", w, 1);
    run<23>("FADD2imm+I2F", w, 2);
    run<24>("REDUX.MAX", w, 1);
  }
  return 0;
}
