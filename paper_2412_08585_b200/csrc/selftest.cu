// selftest.cu -- exhaustive on-device check of the fast correctly-rounded
// divisions of common.cuh (div_by_119, div_119_by) against __fdiv_rn.
#include "common.cuh"

namespace ta {

__global__ void selftest_div_kernel(int which, uint32_t lo, uint32_t hi, unsigned long long* bad, uint32_t* first) {
  const uint64_t n = (uint64_t)hi - lo + 1;
  unsigned long long mine = 0;
  uint32_t fb = 0xFFFFFFFFu;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t bits = lo + (uint32_t)i;
    const float a = __uint_as_float(bits);
    const float fast = which == 0 ? div_by_119(a) : div_119_by(a);
    const float ref = which == 0 ? __fdiv_rn(a, kDiv) : __fdiv_rn(kDiv, a);
    if (__float_as_uint(fast) != __float_as_uint(ref)) {
      ++mine;
      fb = min(fb, bits);
    }
  }
  if (mine) {
    atomicAdd(bad, mine);
    atomicMin(first, fb);
  }
}

}  // namespace ta

namespace ta_host {
cudaError_t launch_selftest_div(int which, uint32_t lo, uint32_t hi, unsigned long long* bad, uint32_t* first,
                                cudaStream_t st) {
  ta::selftest_div_kernel<<<148 * 8, 256, 0, st>>>(which, lo, hi, bad, first);
  return cudaGetLastError();
}
}  // namespace ta_host
