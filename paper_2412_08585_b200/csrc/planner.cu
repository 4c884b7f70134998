// planner.cu -- head-wise mixed precision (Sec. 3.2): per
// (kv_head, K/V) slot priority = gap x std of the channel gaps over the prefill
// tokens, and the n_h lowest-priority slots get 2 bits (R-8).
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace ta {

// Monotone float <-> int map for atomicMax / atomicMin on floats.
TA_DEV int ford(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
TA_DEV float iford(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF); }

// grid (2 Hkv slots, chunks); per channel max/min over the chunk's tokens of
// all batch entries, merged with atomics into ws[slot][d][2] (ordered ints).
template <int HD>
__global__ void __launch_bounds__(256) channel_range_kernel(const __half* __restrict__ k, const __half* __restrict__ v,
                                                            int B, int N, int Hkv, int* __restrict__ ws) {
  constexpr int STRIPES = 256 / HD;
  __shared__ float smax[STRIPES][HD], smin[STRIPES][HD];
  const int slot = blockIdx.x, h = slot >> 1, kind = slot & 1;
  const int c = threadIdx.x % HD, stripe = threadIdx.x / HD;
  const long total = (long)B * N;
  const long per = (total + gridDim.y - 1) / gridDim.y;
  const long t0 = blockIdx.y * per, t1 = min(total, t0 + per);
  const __half* src = kind ? v : k;
  float mx = -INFINITY, mn = INFINITY;
  for (long t = t0 + stripe; t < t1; t += STRIPES) {
    const float x = __half2float(src[(t * Hkv + h) * HD + c]);  // t = b * N + token
    mx = fmaxf(mx, x);
    mn = fminf(mn, x);
  }
  smax[stripe][c] = mx;
  smin[stripe][c] = mn;
  __syncthreads();
  if (stripe == 0) {
#pragma unroll
    for (int s = 1; s < STRIPES; ++s) {
      mx = fmaxf(mx, smax[s][c]);
      mn = fminf(mn, smin[s][c]);
    }
    if (t0 < t1) {
      atomicMax(&ws[(slot * HD + c) * 2 + 0], ford(mx));
      atomicMin(&ws[(slot * HD + c) * 2 + 1], ford(mn));
    }
  }
}

__global__ void range_init_kernel(int* ws, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ws[i] = (i & 1) ? 0x7FFFFFFF : (int)0x80000000;
}

// priority[slot] = (max_c max - min_c min) * population std of (max_c - min_c).
template <int HD>
__global__ void priority_kernel(const int* __restrict__ ws, double* __restrict__ priority) {
  __shared__ double red[4][HD];
  const int slot = blockIdx.x, c = threadIdx.x;
  const float mx = iford(ws[(slot * HD + c) * 2 + 0]), mn = iford(ws[(slot * HD + c) * 2 + 1]);
  const double gap = (double)mx - (double)mn;
  red[0][c] = mx;
  red[1][c] = mn;
  red[2][c] = gap;
  __syncthreads();
  if (c == 0) {
    double gmax = -INFINITY, gmin = INFINITY, mean = 0.0;
    for (int i = 0; i < HD; ++i) {
      gmax = fmax(gmax, red[0][i]);
      gmin = fmin(gmin, red[1][i]);
      mean += red[2][i];
    }
    mean /= HD;
    double var = 0.0;
    for (int i = 0; i < HD; ++i) var += (red[2][i] - mean) * (red[2][i] - mean);
    var /= HD;
    priority[slot] = (gmax - gmin) * sqrt(var);
  }
}

}  // namespace ta

namespace ta_host {
using namespace ta;

size_t priority_workspace(int Hkv, int HD) { return (size_t)2 * Hkv * HD * 2 * sizeof(int); }

cudaError_t launch_priority(int B, int N, int Hkv, int HD, const __half* k, const __half* v, void* ws,
                            double* priority, cudaStream_t st) {
  int* w = reinterpret_cast<int*>(ws);
  const int n = 2 * Hkv * HD * 2;
  range_init_kernel<<<(n + 255) / 256, 256, 0, st>>>(w, n);
  const int chunks = std::max(1, std::min(256, (int)(((long)B * N + 511) / 512)));
  const dim3 grid(2 * Hkv, chunks);
  if (HD == 128) {
    channel_range_kernel<128><<<grid, 256, 0, st>>>(k, v, B, N, Hkv, w);
    priority_kernel<128><<<2 * Hkv, 128, 0, st>>>(w, priority);
  } else {
    channel_range_kernel<64><<<grid, 256, 0, st>>>(k, v, B, N, Hkv, w);
    priority_kernel<64><<<2 * Hkv, 64, 0, st>>>(w, priority);
  }
  return cudaGetLastError();
}

// Rank the slots by priority (ties toward the lower slot index) and give the
// n_2bit lowest 2 bits, the rest 4.  Host-side, 2 Hkv values.
void plan_bits(const double* priority, int n_slots, int n_2bit, int32_t* bits) {
  std::vector<int> order(n_slots);
  for (int i = 0; i < n_slots; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return priority[a] < priority[b]; });
  for (int i = 0; i < n_slots; ++i) bits[i] = 4;
  for (int i = 0; i < n_2bit && i < n_slots; ++i) bits[order[i]] = 2;
}
}  // namespace ta_host
