"""Python (ctypes + numpy) front end of the CPU oracle in ``turbo_oracle.c``.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  It shares no code with the CUDA path (``paper_2412_08585_b200``) and
never imports it; inputs come from ``paper_2412_08585_b200.synth`` (seeded
generators that hold none of the method's arithmetic) or from the tests.

Every function mirrors one routine of the paper (citations in turbo_oracle.c):
Alg. 1 prefill and its chunked form (reading R-28), Alg. 2 decode
(PAPER.md:945-997), SAS
(PAPER.md:455-493, 1006-1032), FlashQ stage 1/2 and the
enhanced KV buffer.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "turbo_oracle.c")
_LIB = os.path.join(_HERE, "_build", "libturbo_oracle.so")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (scalar, no fast-math, no FMA contraction).

    ``TURBO_ORACLE_LIB`` names a prebuilt library instead (used only by
    tests/test_oracle_mutations.py to load deliberately broken oracles)."""
    if os.environ.get("TURBO_ORACLE_LIB"):
        return os.environ["TURBO_ORACLE_LIB"]
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "turbo_oracle.h"))
    ):
        os.makedirs(os.path.dirname(_LIB), exist_ok=True)
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _declare(_lib)
    return _lib


class Params(C.Structure):
    _fields_ = [
        ("d", C.c_int32), ("block_q", C.c_int32), ("block_kv", C.c_int32), ("sas_nr", C.c_int32),
        ("alpha_mode", C.c_int32), ("softmax_scale", C.c_float), ("quant", C.c_int32), ("sas", C.c_int32),
        ("p_row", C.c_int32),
        ("scale_fp16", C.c_int32), ("sas_fp16", C.c_int32),
    ]


class _Slot(C.Structure):
    _fields_ = [
        ("bits", C.c_int32), ("max_blocks", C.c_int32), ("n_blocks", C.c_int32), ("n_buf", C.c_int32),
        ("codes", C.c_void_p), ("s_int", C.c_void_p), ("z_int", C.c_void_p), ("s_parent", C.c_void_p),
        ("buf", C.c_void_p), ("a_univ", C.c_float),
    ]


class _PrefillTap(C.Structure):
    _fields_ = [("i_block", C.c_int32), ("j_block", C.c_int32), ("hit", C.c_int32)] + [
        (n, C.c_void_p) for n in ("q1", "s_q", "s_int", "m_new", "p_tilde", "p_codes", "s_p", "pv_int")
    ]


class _DecodeTap(C.Structure):
    _fields_ = [("j_block", C.c_int32), ("hit", C.c_int32)] + [
        (n, C.c_void_p) for n in ("q1", "s_q", "s_int", "m_new", "p_tilde", "p_codes", "s_p", "pv_int")
    ]


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _declare(L):
    vp, i32, i64, f32 = C.c_void_p, C.c_int32, C.c_int64, C.c_float
    L.tq_sas_lut.argtypes = [i32, vp]
    L.tq_sas_poly.argtypes = [f32]
    L.tq_sas_poly.restype = f32
    L.tq_sas.argtypes = [f32, i32]
    L.tq_sas.restype = f32
    L.tq_sas_poly_fp16.argtypes = [f32]
    L.tq_sas_poly_fp16.restype = f32
    L.tq_sas_fp16.argtypes = [f32, i32]
    L.tq_sas_fp16.restype = f32
    L.tq_sas_softmax_rows.argtypes = [i32, i32, vp, i32, vp]
    L.tq_quant_sym8.argtypes = [vp, i64, vp, vp]
    L.tq_quant_asym.argtypes = [vp, i32, i64, i32, vp, i64, vp, vp]
    L.tq_dequant_q2.argtypes = [i32, i32, i32]
    L.tq_dequant_q2.restype = i32
    L.tq_cache_prefill_slot.argtypes = [C.POINTER(Params), i32, vp, C.POINTER(_Slot), vp, vp]
    L.tq_cache_prefill_slot.restype = i32
    L.tq_cache_append_slot.argtypes = [C.POINTER(Params), vp, C.POINTER(_Slot)]
    L.tq_cache_append_slot.restype = i32
    L.tq_cache_prefill_append_slot.argtypes = [C.POINTER(Params), i32, vp, C.POINTER(_Slot), vp, vp]
    L.tq_cache_prefill_append_slot.restype = i32
    L.tq_prefill_chunk_head.argtypes = [C.POINTER(Params), i32, i32, i32, vp, vp, vp, vp, vp, vp, vp]
    L.tq_prefill_chunk_head.restype = i32
    L.tq_prefill_head.argtypes = [C.POINTER(Params), i32, i32, vp, vp, vp, vp, vp, vp]
    L.tq_prefill_head.restype = i32
    L.tq_prefill_head_blocks.argtypes = [C.POINTER(Params), i32, i32, vp, vp, vp, i32, i32, vp, vp, vp]
    L.tq_prefill_head_blocks.restype = i32
    L.tq_decode_head.argtypes = [C.POINTER(Params), vp, C.POINTER(_Slot), C.POINTER(_Slot), vp, vp, i32,
                                 i32, i32, i32, vp, vp, vp]
    L.tq_decode_head.restype = i32
    L.tq_combine.argtypes = [i32, i32, vp, vp, vp, vp]
    L.tq_reference_attention.argtypes = [i32, i32, i32, vp, vp, vp, i32, i32, C.c_double, vp, vp]
    L.tq_head_priority.argtypes = [i32, i32, vp, vp]
    L.tq_slot_univ_scale.argtypes = [vp, vp]
    L.tq_slot_univ_scale.restype = f32


def params(d=128, block_q=64, block_kv=64, sas_nr=-6, alpha_mode=0, softmax_scale=None, quant=1, sas=1, p_row=0,
           scale_fp16=0, sas_fp16=0):
    """Paper defaults: B_r = B_c = n_b = 64, n_r = -6; p_row=1 is the
    per-row prefill P scale, scale_fp16=1 FP16 first-stage scales, sas_fp16=1 the FP16 SAS
    polynomial (NEXT-2 variants)."""
    if softmax_scale is None:
        softmax_scale = float(np.float32(1.0) / np.sqrt(np.float32(d)))
    return Params(d, block_q, block_kv, sas_nr, alpha_mode, softmax_scale, quant, sas, p_row, scale_fp16, sas_fp16)


def _f32(x):
    return np.ascontiguousarray(x, dtype=np.float32)


# ---------------------------------------------------------------- SAS
def sas_lut(nr=-6) -> np.ndarray:
    out = np.zeros(-nr + 1, np.float32)
    lib().tq_sas_lut(nr, _p(out))
    return out


def sas_poly(f: float) -> np.float32:
    return np.float32(lib().tq_sas_poly(float(f)))


def sas(dist: float, nr=-6) -> np.float32:
    return np.float32(lib().tq_sas(float(np.float32(dist)), nr))


def sas_poly_fp16(f: float) -> np.float32:
    return np.float32(lib().tq_sas_poly_fp16(float(np.float32(f))))


def sas_fp16(dist: float, nr=-6) -> np.float32:
    return np.float32(lib().tq_sas_fp16(float(np.float32(dist)), nr))


def sas_softmax_rows(x: np.ndarray, nr=-6) -> np.ndarray:
    x = _f32(np.atleast_2d(x))
    out = np.empty_like(x)
    lib().tq_sas_softmax_rows(x.shape[0], x.shape[1], _p(x), nr, _p(out))
    return out


# ---------------------------------------------------------------- FlashQ
def quant_sym8(x: np.ndarray):
    x = _f32(x)
    codes = np.empty(x.shape, np.int8)
    s = np.zeros(1, np.float32)
    lib().tq_quant_sym8(_p(x), x.size, _p(codes), _p(s))
    return codes, np.float32(s[0])


def quant_asym(g: np.ndarray, bits: int):
    g = np.ascontiguousarray(g, dtype=np.int8)
    codes = np.empty(g.shape, np.uint8)
    s = np.zeros(1, np.uint8)
    z = np.zeros(1, np.int8)
    lib().tq_quant_asym(_p(g), g.size, 1, bits, _p(codes), 1, _p(s), _p(z))
    return codes, int(s[0]), int(z[0])


def dequant_q2(code, s_int, z_int) -> int:
    return lib().tq_dequant_q2(int(code), int(s_int), int(z_int))


# ---------------------------------------------------------------- cache
@dataclass
class Slot:
    """One (batch, kv_head, K-or-V) cache stream, logical (unpacked) layout."""
    p: Params
    bits: int
    max_blocks: int
    codes: np.ndarray = field(init=False)
    s_int: np.ndarray = field(init=False)
    z_int: np.ndarray = field(init=False)
    s_parent: np.ndarray = field(init=False)
    buf: np.ndarray = field(init=False)
    c: _Slot = field(init=False)

    def __post_init__(self):
        d, bc = self.p.d, self.p.block_kv
        self.codes = np.zeros((self.max_blocks, bc, d), np.uint8)
        self.s_int = np.zeros((self.max_blocks, d), np.uint8)
        self.z_int = np.zeros((self.max_blocks, d), np.int8)
        self.s_parent = np.zeros(self.max_blocks, np.float32)
        self.buf = np.zeros((bc, d), np.int8)
        self.c = _Slot(self.bits, self.max_blocks, 0, 0, _p(self.codes), _p(self.s_int), _p(self.z_int),
                       _p(self.s_parent), _p(self.buf), 0.0)

    @property
    def n_blocks(self):
        return self.c.n_blocks

    @property
    def n_buf(self):
        return self.c.n_buf

    @property
    def a_univ(self):
        return np.float32(self.c.a_univ)

    def prefill(self, x: np.ndarray):
        """Returns (x1 [N][d] int8, x1_scale [T_c] f32): the stage-1 prefill operands."""
        x = _f32(x)
        n = x.shape[0]
        tc = -(-n // self.p.block_kv)
        x1 = np.zeros((n, self.p.d), np.int8)
        sc = np.zeros(tc, np.float32)
        rc = lib().tq_cache_prefill_slot(C.byref(self.p), n, _p(x), C.byref(self.c), _p(x1), _p(sc))
        if rc != 0:
            raise ValueError(f"tq_cache_prefill_slot -> {rc}")
        return x1, sc

    def prefill_append(self, x: np.ndarray):
        """A further prefill chunk (R-28; R-31 when the cache ends inside a block): returns the
        chunk's stage-1 operands (x1 [n][d] int8, x1_scale f32 of the chunk's own blocks -- the
        boundary block's scale s_univ belongs to stage1_prefix(with_buffer=True))."""
        x = _f32(x)
        n = x.shape[0]
        bc = self.p.block_kv
        r = min(n, bc - self.n_buf) if self.n_buf else 0
        tc = -(-(n - r) // bc)
        x1 = np.zeros((n, self.p.d), np.int8)
        sc = np.zeros(tc, np.float32)
        rc = lib().tq_cache_prefill_append_slot(C.byref(self.p), n, _p(x), C.byref(self.c), _p(x1), _p(sc))
        if rc != 0:
            raise ValueError(f"tq_cache_prefill_append_slot -> {rc}")
        return x1, sc

    def stage1_prefix(self, n_blocks: int, with_buffer: bool = False):
        """Stage-1 reconstruction of blocks [0, n_blocks): int8 [n_blocks B_c][d] codes
        code s^int + z^int (Alg. 2) with the blocks' parent scales; with_buffer: then
        the n_buf buffered tokens' codes and the boundary block's scale s_univ (R-31)."""
        x1 = np.concatenate([self.dequant_block(j) for j in range(n_blocks)], 0) if n_blocks else \
            np.zeros((0, self.p.d), np.int32)
        sc = self.s_parent[:n_blocks].copy()
        if with_buffer and self.n_buf:
            x1 = np.concatenate([x1, self.buf[:self.n_buf].astype(np.int32)], 0)
            sc = np.concatenate([sc, [np.float32(lib().tq_slot_univ_scale(C.byref(self.p), C.byref(self.c)))]])
        return x1.astype(np.int8), sc.astype(np.float32)

    def append(self, x: np.ndarray):
        x = _f32(x)
        rc = lib().tq_cache_append_slot(C.byref(self.p), _p(x), C.byref(self.c))
        if rc != 0:
            raise ValueError(f"tq_cache_append_slot -> {rc}")

    def dequant_block(self, j: int) -> np.ndarray:
        """K^q1 = K^q2 s^int + z^int for block j (int, [B_c][d])."""
        return self.codes[j].astype(np.int32) * self.s_int[j].astype(np.int32) + self.z_int[j].astype(np.int32)


# ---------------------------------------------------------------- attention
def _tap_arrays(rows, bc, d):
    return dict(q1=np.zeros((rows, d), np.int8), s_q=np.zeros(1, np.float32),
                s_int=np.zeros((rows, bc), np.int32), m_new=np.zeros(rows, np.float32),
                p_tilde=np.zeros((rows, bc), np.float32), p_codes=np.zeros((rows, bc), np.uint8),
                s_p=np.zeros(1, np.float32), pv_int=np.zeros((rows, d), np.int32))


def prefill_head(p: Params, q, k, v, causal=True, tap=None, blocks=None):
    """Alg. 1 for one (batch, head): q, k, v [N][d] (fp16-valued floats).

    Returns (O [N][d] f32, L [N] f32[, tap dict]).  ``tap=(i, j)`` records the
    exact-set intermediates of B_r block i x KV block j.  ``blocks=(i0, i1)``
    runs only query blocks i0 <= i < i1 of the (independent) outer loop; the
    other rows stay zero.
    """
    q, k, v = _f32(q), _f32(k), _f32(v)
    n = q.shape[0]
    o = np.zeros((n, p.d), np.float32)
    lse = np.zeros(n, np.float32)
    t = None
    if tap is not None:
        arrs = _tap_arrays(p.block_q, p.block_kv, p.d)
        t = _PrefillTap(tap[0], tap[1], 0, *[_p(arrs[k_]) for k_ in
                                             ("q1", "s_q", "s_int", "m_new", "p_tilde", "p_codes", "s_p", "pv_int")])
    i0, i1 = blocks if blocks is not None else (0, 2**31 - 1)
    rc = lib().tq_prefill_head_blocks(C.byref(p), n, int(causal), _p(q), _p(k), _p(v), i0, i1, _p(o), _p(lse),
                                      C.byref(t) if t is not None else None)
    if rc != 0:
        raise ValueError(f"tq_prefill_head -> {rc}")
    if tap is not None:
        arrs["hit"] = bool(t.hit)
        return o, lse, arrs
    return o, lse


def prefill_chunk_head(p: Params, q, k1, sk, v1, sv, causal=True):
    """Chunked prefill (R-28): Alg. 1 for the nq rows of q at positions nk - nq ..
    nk - 1 against nk keys given as stage-1 operands k1, v1 (int8 [nk][d]) with
    block scales sk, sv.  Returns (O [nq][d] f32, L [nq] f32)."""
    q = _f32(q)
    k1, v1 = np.ascontiguousarray(k1, np.int8), np.ascontiguousarray(v1, np.int8)
    sk, sv = _f32(sk), _f32(sv)
    nq, nk = q.shape[0], k1.shape[0]
    o = np.zeros((nq, p.d), np.float32)
    lse = np.zeros(nq, np.float32)
    rc = lib().tq_prefill_chunk_head(C.byref(p), nq, nk, int(causal), _p(q), _p(k1), _p(sk), _p(v1), _p(sv),
                                     _p(o), _p(lse))
    if rc != 0:
        raise ValueError(f"tq_prefill_chunk_head -> {rc}")
    return o, lse


def decode_head(p: Params, q, kslot: Slot | None, vslot: Slot | None, blk_begin=0, blk_end=None,
                with_buffer=True, k_raw=None, v_raw=None, tap=None):
    """Alg. 2 for one query head against one (b, kv_head) cache; returns (O f32 [d], L)."""
    q = _f32(q)
    if blk_end is None:
        blk_end = kslot.n_blocks
    o = np.zeros(p.d, np.float32)
    lse = np.zeros(1, np.float32)
    kr = _f32(k_raw) if k_raw is not None else np.zeros((1, p.d), np.float32)
    vr = _f32(v_raw) if v_raw is not None else np.zeros((1, p.d), np.float32)
    n_raw = kr.shape[0] if k_raw is not None else 0
    t = None
    if tap is not None:
        arrs = {k_: v_[0] if v_.ndim == 2 else v_ for k_, v_ in _tap_arrays(1, p.block_kv, p.d).items()}
        arrs = {k_: np.ascontiguousarray(v_) for k_, v_ in arrs.items()}
        t = _DecodeTap(tap, 0, *[_p(arrs[k_]) for k_ in
                                 ("q1", "s_q", "s_int", "m_new", "p_tilde", "p_codes", "s_p", "pv_int")])
    rc = lib().tq_decode_head(C.byref(p), _p(q), C.byref(kslot.c), C.byref(vslot.c), _p(kr), _p(vr), n_raw,
                              blk_begin, blk_end, int(with_buffer), _p(o), _p(lse),
                              C.byref(t) if t is not None else None)
    if rc != 0:
        raise ValueError(f"tq_decode_head -> {rc}")
    if tap is not None:
        arrs["hit"] = bool(t.hit)
        return o, np.float32(lse[0]), arrs
    return o, np.float32(lse[0])


def combine(o_parts: np.ndarray, lse_parts: np.ndarray):
    o_parts = _f32(o_parts)
    lse_parts = _f32(lse_parts)
    n, d = o_parts.shape
    o = np.zeros(d, np.float32)
    lse = np.zeros(1, np.float32)
    lib().tq_combine(n, d, _p(o_parts), _p(lse_parts), _p(o), _p(lse))
    return o, np.float32(lse[0])


def reference_attention(q, k, v, causal=True, q_offset=0, scale=None):
    """Eq. 2 in float64 (brute force, the exact-attention reference)."""
    q = np.ascontiguousarray(q, np.float64)
    k = np.ascontiguousarray(k, np.float64)
    v = np.ascontiguousarray(v, np.float64)
    nq, d = q.shape
    nk = k.shape[0]
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    o = np.zeros((nq, d))
    lse = np.zeros(nq)
    lib().tq_reference_attention(nq, nk, d, _p(q), _p(k), _p(v), int(causal), q_offset, float(scale),
                                 _p(o), _p(lse))
    return o, lse


def head_priority(x: np.ndarray) -> float:
    x = _f32(x)
    out = np.zeros(1, np.float64)
    lib().tq_head_priority(x.shape[0], x.shape[1], _p(x), _p(out))
    return float(out[0])


def plan_bits(priorities, n_2bit: int) -> np.ndarray:
    """Head-wise mixed precision: the n_h lowest-priority
    slots get 2 bits, the rest 4; ties resolved toward the lower slot index."""
    pr = np.asarray(priorities, np.float64)
    order = sorted(range(len(pr)), key=lambda i: (pr[i], i))
    bits = np.full(len(pr), 4, np.int32)
    bits[order[:n_2bit]] = 2
    return bits


# ---------------------------------------------------------------- whole-tensor helpers
def project_q(x, wq):
    """The FP16 output of the Q projection: Q = fp16(x wq^T) with the product
    formed in float64 and rounded once to binary16 (nearest even) -- a library matmul as one
    step.  x [..., D], wq [Hq d][D] -> [..., Hq d] float16."""
    return (np.asarray(x, np.float64) @ np.asarray(wq, np.float64).T).astype(np.float16)


def build_cache(p: Params, k, v, bits, max_blocks):
    """Cache for a [B][N][Hkv][d] K/V pair: returns dict with slots[b][h] = (Kslot, Vslot),
    and the stage-1 prefill operands k1/v1 [B][Hkv][N][d], k1s/v1s [B][Hkv][T_c]."""
    B, N, H, d = k.shape
    tc = -(-N // p.block_kv)
    out = dict(slots=[[None] * H for _ in range(B)], k1=np.zeros((B, H, N, d), np.int8),
               v1=np.zeros((B, H, N, d), np.int8), k1s=np.zeros((B, H, tc), np.float32),
               v1s=np.zeros((B, H, tc), np.float32))
    for b in range(B):
        for h in range(H):
            ks = Slot(p, int(bits[h][0]), max_blocks)
            vs = Slot(p, int(bits[h][1]), max_blocks)
            out["k1"][b, h], out["k1s"][b, h] = ks.prefill(k[b, :, h])
            out["v1"][b, h], out["v1s"][b, h] = vs.prefill(v[b, :, h])
            out["slots"][b][h] = (ks, vs)
    return out
