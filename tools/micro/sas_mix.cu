// Throughput of the prefill softmax's pass-2 instruction mix in isolation: the bit-exact SAS of
// 64 register-resident scores per thread (FADD2 d, FADD2.RM floor, FADD2 x2 frac, SHFL LUT x2,
// FFMA2 x3 Horner, FMUL2 LUT product, FSETP/FSEL threshold, FADD2 row sum, FMNMX max) with no
// TMEM, no barriers -- W warps per SM, one CTA per SM.  Prints score elements per clock per SM
// (the prefill at 604 TOPS runs ~4.1 elements/clk/SM through all three passes).
#include <cstdio>
#include "common.cuh"

using namespace ta;

template <int NW, int V>
__global__ void __launch_bounds__(32 * NW, 1) kern(int iters, float seed, unsigned long long* cyc, float* sink) {
  const int lane = threadIdx.x & 31;
  const float lut_lane = lane <= 6 ? __uint_as_float(kExpNegBits[lane]) : 0.f;
  uint32_t v[64];
#pragma unroll
  for (int c = 0; c < 64; ++c) v[c] = __float_as_uint(seed * (float)((c * 37 + threadIdx.x) % 97) * 0.07f);
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (V & 4) {  // pass 1: int S -> x = S c, row max
      const f32x2 cq2 = pk2(seed, seed);
      float mt = -INFINITY, mt1 = -INFINITY;
#pragma unroll
      for (int c = 0; c < 64; c += 4) {
        const f32x2 x2 = mul2(pk2((float)(int)v[c], (float)(int)v[c + 1]), cq2);
        const f32x2 y2 = mul2(pk2((float)(int)v[c + 2], (float)(int)v[c + 3]), cq2);
        mt = fmaxf(mt, fmaxf(lo2(x2), hi2(x2)));
        mt1 = fmaxf(mt1, fmaxf(lo2(y2), hi2(y2)));
        v[c] = __float_as_uint(lo2(x2));
        v[c + 1] = __float_as_uint(hi2(x2));
        v[c + 2] = __float_as_uint(lo2(y2));
        v[c + 3] = __float_as_uint(hi2(y2));
      }
      acc += fmaxf(mt, mt1);
    }
    const float m_use = __uint_as_float(v[it & 63]) + 1.f;
    float pmax = 0.f, pmax1 = 0.f;
    f32x2 rs[4] = {pk2(0.f, 0.f), pk2(0.f, 0.f), pk2(0.f, 0.f), pk2(0.f, 0.f)};
    const f32x2 m2 = pk2(m_use, m_use), mg2 = pk2(kMagic, kMagic);
    const f32x2 c3 = pk2(-0.1025f, -0.1025f), c2 = pk2(0.4626f, 0.4626f), c1 = pk2(-0.9922f, -0.9922f),
                c0 = pk2(0.9996f, 0.9996f);
#pragma unroll
    for (int c = 0; c < 64; c += 2) {
      const f32x2 d2 = sub2(m2, pk2(__uint_as_float(v[c]), __uint_as_float(v[c + 1])));
      const f32x2 t2 = add2_rd(d2, mg2);
      const f32x2 f2 = sub2(d2, sub2(t2, mg2));
      const float l0 = (V & 1) ? __uint_as_float(__float_as_uint(lut_lane) ^ (__float_as_uint(lo2(t2)) & 7u))
                               : lut_shfl(lut_lane, __float_as_uint(lo2(t2)));
      const float l1 = (V & 1) ? __uint_as_float(__float_as_uint(lut_lane) ^ (__float_as_uint(hi2(t2)) & 7u))
                               : lut_shfl(lut_lane, __float_as_uint(hi2(t2)));
      const f32x2 p2 = fma2(fma2(fma2(c3, f2, c2), f2, c1), f2, c0);
      const f32x2 lp = mul2(pk2(l0, l1), p2);
      const float pt0 = (V & 2) ? lo2(lp) : (lo2(d2) > 6.f ? 0.f : lo2(lp));
      const float pt1 = (V & 2) ? hi2(lp) : (hi2(d2) > 6.f ? 0.f : hi2(lp));
      rs[(c >> 1) & 3] = add2(rs[(c >> 1) & 3], pk2(pt0, pt1));
      if (c & 2) pmax1 = fmaxf(pmax1, fmaxf(pt0, pt1));
      else pmax = fmaxf(pmax, fmaxf(pt0, pt1));
      v[c] = __float_as_uint(__uint_as_float(v[c]) + pt0);  // feed back (keeps the work live)
      v[c + 1] = __float_as_uint(__uint_as_float(v[c + 1]) + pt1);
    }
    const f32x2 r = add2(add2(rs[0], rs[1]), add2(rs[2], rs[3]));
    acc += lo2(r) + hi2(r) + fmaxf(pmax, pmax1);
    if (V & 4) {  // pass 3: P codes (magic FFMA2), fp16 pack (PRMT), P' hi / lo (2 HFMA2)
      const f32x2 inv2 = pk2(acc, acc), mf2 = pk2(12582912.0f + 25600.0f, 12582912.0f + 25600.0f);
      uint32_t hsum = 0;
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const f32x2 y2 = fma2(pk2(__uint_as_float(v[2 * e]), __uint_as_float(v[2 * e + 1])), inv2, mf2);
        const uint32_t y = __byte_perm(__float_as_uint(lo2(y2)), __float_as_uint(hi2(y2)), 0x5410);
        const uint32_t ph = hfma2_u32(y, 0x3c003c00u, 0xe400e400u), pl = hfma2_u32(y, 0x1c001c00u, 0x84008400u);
        v[2 * e] = ph;
        v[2 * e + 1] = pl;
        hsum ^= ph ^ pl;
      }
      acc += (float)hsum;
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc + __uint_as_float(v[threadIdx.x & 63]);
}

template <int NW, int V>
void run() {
  unsigned long long* cyc;
  float* sink;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&sink, 148 * 1024 * 4);
  const int iters = 2000;
  kern<NW, V><<<148, 32 * NW>>>(16, 1.f, cyc, sink);
  cudaMemset(cyc, 0, 8);
  kern<NW, V><<<148, 32 * NW>>>(iters, 1.f, cyc, sink);
  unsigned long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double clk = (double)h / 148;
  const double elems = (double)iters * 64 * 32 * NW;
  printf("pass-2 mix V%d (%s%s), %2d warps/SM: %.2f elements/clk/SM\n", V, (V & 1) ? "no SHFL " : "",
         (V & 2) ? "no threshold" : "", NW, elems / clk);
  if (V & 4) printf("   (V4 = all three passes: pass 1 + pass 2 + pass 3 per element)\n");
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  run<4, 0>();
  run<8, 0>();
  run<12, 0>();
  run<4, 4>();
  run<8, 4>();
  run<12, 4>();
  run<4, 1>();
  run<8, 1>();
  run<4, 2>();
  run<8, 2>();
  run<4, 3>();
  run<8, 3>();
  return 0;
}
