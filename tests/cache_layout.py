"""Decoder of the GPU cache's packed block records (written from
that documented byte layout) into the oracle's logical [token][channel] codes.
Test-side only; shares no code with the CUDA path or the oracle.

A B_c = 128 block stores its V codes as two 64-token sub-blocks back to back,
each in the 64-token channel-major layout."""
import numpy as np

BC = 64   # default block size; every function takes bc=
SUB = 64  # V code sub-block (tokens)


def unpack_k(codes_bytes: np.ndarray, d: int, bits: int, bc: int = BC) -> np.ndarray:
    """K: token-major, natural channel order, LSB-first within each byte."""
    per = 8 // bits
    tb = d * bits // 8
    raw = codes_bytes[: bc * tb].reshape(bc, tb)
    out = np.zeros((bc, d), np.uint8)
    for i in range(per):
        out[:, i::per] = (raw >> (bits * i)) & ((1 << bits) - 1)
    return out


def v_token(bits: int, wi: int, i: int):
    """(token, byte e, bit shift) of code i in V word wi of a 64-token sub-block (layout.cuh)."""
    if bits == 4:
        j, q, nib = wi >> 2, wi & 3, i & 1
        e = i >> 1
        return 32 * j + 16 * nib + 4 * q + e, e, 4 * nib
    q, s = wi, i & 3
    e = i >> 2
    return 32 * (s >> 1) + 16 * (s & 1) + 4 * q + e, e, 2 * s


def unpack_v(codes_bytes: np.ndarray, d: int, bits: int, bc: int = BC) -> np.ndarray:
    cb = SUB * bits // 8  # bytes per channel per sub-block
    out = np.zeros((bc, d), np.uint8)
    for u in range(bc // SUB):
        part = np.ascontiguousarray(codes_bytes[u * d * cb:(u + 1) * d * cb])
        words = part.view(np.uint32).reshape(d, cb // 4)
        for wi in range(cb // 4):
            for i in range(32 // bits):
                t, e, sh = v_token(bits, wi, i)
                out[SUB * u + t, :] = (words[:, wi] >> (8 * e + sh)) & ((1 << bits) - 1)
    return out


def unpack_record(rec: np.ndarray, d: int, bits: int, kind: int, bc: int = BC):
    s_int = rec[:d].copy()
    z_int = rec[d:2 * d].view(np.int8).copy()
    codes = (unpack_k if kind == 0 else unpack_v)(rec[2 * d:], d, bits, bc)
    return codes, s_int, z_int
