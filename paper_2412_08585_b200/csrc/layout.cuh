// layout.cuh -- byte layout of a stage-2 block record.
//
// record = s_int u8[d] | z_int i8[d] | codes, rec_bytes = 2d + B_c d / 2
// (B_c in {64, 128}; 2-bit blocks use the first half of the code area).
//
// K codes (token-major, natural channel order; LSB-first): token t occupies
//   d*bits/8 bytes; byte b holds channels b*8/bits ... (b+1)*8/bits - 1.
//   The decode kernel gives lane quad q the contiguous channel region
//   [q d/4, (q+1) d/4) of a token and maps mma k-slots onto it (decode.cu).
//
// V codes (channel-major per 64-token sub-block): sub-block u (tokens
//   64u .. 64u + 63; one sub-block when B_c = 64, two when B_c = 128) occupies
//   d * 64*bits/8 bytes, channel c of it 64*bits/8 bytes of 32-bit words
//   (the token indices below are relative to the sub-block).  The token order inside a channel matches the mma.sync m16n8k32
//   A-fragment of V^T (rows = channels, k = tokens), so one 32-bit load plus
//   a mask/shift gives a ready fragment register:
//     4-bit: word W = 4j + q (k-step j in {0,1}, quad q): byte e holds token
//            32j + 4q + e (low nibble) and token 32j + 16 + 4q + e (high nibble).
//     2-bit: word q: byte e, bits [2s, 2s+2) hold token
//            32*(s>>1) + 16*(s&1) + 4q + e   (s = 0..3).
#pragma once
#include "common.cuh"

namespace ta {

__host__ __device__ constexpr int rec_bytes(int hd, int bc = kBc) { return 2 * hd + bc * hd / 2; }
constexpr int kSub = 64;  // V code sub-block (tokens)

// Token stored at code index i (0 .. 32/bits - 1) of V word wi; returns the
// token and sets the byte e and bit shift sh inside that byte.
__host__ __device__ inline int v_token_of(int bits, int wi, int i, int* e, int* sh) {
  if (bits == 4) {
    const int j = wi >> 2, q = wi & 3, nib = i & 1;
    *e = i >> 1;
    *sh = 4 * nib;
    return 32 * j + 16 * nib + 4 * q + *e;
  } else {
    const int q = wi, s = i & 3;
    *e = i >> 2;
    *sh = 2 * s;
    return 32 * (s >> 1) + 16 * (s & 1) + 4 * q + *e;
  }
}

}  // namespace ta
