"""Thin ctypes binding of libturboattn.so (include/turbo_attention.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels behind the C-ABI.  PyTorch provides device memory and the stream.
There is no CPU fallback -- if the library is missing or the GPU is not an
sm_100 part, calls raise.
"""
from __future__ import annotations

import ctypes as C
import math
import os

import torch

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TURBO_LIB", os.path.join(PKG, "libturboattn.so"))

TURBO_OK, TURBO_ERR_INVALID_ARG, TURBO_ERR_UNSUPPORTED, TURBO_ERR_CAPACITY, TURBO_ERR_CUDA = range(5)
_ERR = {1: "TURBO_ERR_INVALID_ARG", 2: "TURBO_ERR_UNSUPPORTED", 3: "TURBO_ERR_CAPACITY", 4: "TURBO_ERR_CUDA"}

EXPORTS = ("turbo_version", "turbo_cache_sizes", "turbo_quantize_kv", "turbo_attention_prefill",
           "turbo_attention_prefill_chunk", "turbo_dequantize_cache", "turbo_q_projection",
           "turbo_attention_prefill_q1",
           "turbo_decode_workspace_bytes", "turbo_decode_workers", "turbo_attention_decode", "turbo_combine_lse",
           "turbo_priority_workspace_bytes", "turbo_head_priority", "turbo_plan_bits", "turbo_selftest_div")


class TurboError(RuntimeError):
    def __init__(self, fn, code):
        super().__init__(f"{fn} -> {_ERR.get(code, code)}")
        self.code = code


class TurboParams(C.Structure):
    _fields_ = [("head_dim", C.c_int32), ("block_q", C.c_int32), ("block_kv", C.c_int32), ("sas_nr", C.c_int32),
                ("alpha_mode", C.c_int32), ("softmax_scale", C.c_float), ("p_scale_rows", C.c_int32),
                ("scale_fp16", C.c_int32), ("sas_fp16", C.c_int32), ("debug_tap", C.c_void_p)]


class TurboKVCache(C.Structure):
    _fields_ = [("batch", C.c_int32), ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("block_kv", C.c_int32),
                ("max_blocks", C.c_int32), ("n_tokens", C.c_int64), ("bits_host", C.c_void_p),
                ("bits_dev", C.c_void_p), ("block_rec", C.c_void_p), ("s_parent", C.c_void_p), ("buf", C.c_void_p),
                ("a_univ", C.c_void_p), ("counters", C.c_void_p)]


class TurboDebugTap(C.Structure):
    _fields_ = [("batch", C.c_int32), ("head", C.c_int32), ("i_block", C.c_int32), ("j_block", C.c_int32),
                ("q1", C.c_void_p), ("s_q", C.c_void_p), ("s_int", C.c_void_p), ("m_new", C.c_void_p),
                ("p_codes", C.c_void_p), ("s_p", C.c_void_p), ("pv_int", C.c_void_p)]


_lib = None


def lib() -> C.CDLL:
    """Load libturboattn.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2412_08585_b200.build`")
        L = C.CDLL(LIB_PATH)
        vp, i32, sz = C.c_void_p, C.c_int32, C.c_size_t
        L.turbo_version.restype = C.c_char_p
        L.turbo_cache_sizes.argtypes = [i32, i32, i32, i32, i32] + [C.POINTER(sz)] * 5
        L.turbo_quantize_kv.argtypes = [C.POINTER(TurboParams), C.POINTER(TurboKVCache), vp, vp, i32, i32, vp, vp,
                                        vp, vp, vp]
        L.turbo_attention_prefill.argtypes = [C.POINTER(TurboParams), i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp,
                                              vp, vp]
        if hasattr(L, "turbo_attention_prefill_chunk"):  # (older A/B builds lack it)
            L.turbo_attention_prefill_chunk.argtypes = [C.POINTER(TurboParams), i32, i32, i32, i32, i32, i32, vp, vp,
                                                        vp, vp, vp, vp, vp, vp]
            L.turbo_dequantize_cache.argtypes = [C.POINTER(TurboParams), C.POINTER(TurboKVCache), i32, i32, vp, vp,
                                                 vp, vp, i32, vp]
        if hasattr(L, "turbo_q_projection"):  # (older A/B builds lack it)
            L.turbo_q_projection.argtypes = [C.POINTER(TurboParams), i32, i32, i32, i32, vp, vp, vp, vp, vp, vp]
            L.turbo_attention_prefill_q1.argtypes = [C.POINTER(TurboParams), i32, i32, i32, i32, i32, vp, vp, vp, vp,
                                                     vp, vp, vp, vp, vp]
        L.turbo_decode_workspace_bytes.argtypes = [i32, i32, i32, i32, i32]
        L.turbo_decode_workspace_bytes.restype = sz
        if hasattr(L, "turbo_decode_workers"):  # (older A/B builds lack it)
            L.turbo_decode_workers.argtypes = [i32, i32, i32]
            L.turbo_decode_workers.restype = i32
        L.turbo_attention_decode.argtypes = [C.POINTER(TurboParams), C.POINTER(TurboKVCache), i32, vp, i32, i32, i32,
                                             i32, vp, sz, vp, vp, vp, vp]
        L.turbo_combine_lse.argtypes = [i32, i32, i32, vp, vp, vp, vp, vp, vp]
        L.turbo_priority_workspace_bytes.argtypes = [i32, i32]
        L.turbo_priority_workspace_bytes.restype = sz
        L.turbo_head_priority.argtypes = [i32, i32, i32, i32, vp, vp, vp, sz, vp, vp]
        L.turbo_plan_bits.argtypes = [vp, i32, i32, vp]
        if hasattr(L, "turbo_selftest_div"):  # self-test entry (absent from older A/B builds in variants/)
            L.turbo_selftest_div.argtypes = [i32, C.c_uint32, C.c_uint32, vp, vp, vp]
            L.turbo_selftest_div.restype = C.c_int
        for name in ("turbo_cache_sizes", "turbo_quantize_kv", "turbo_attention_prefill", "turbo_attention_decode",
                     "turbo_combine_lse", "turbo_head_priority", "turbo_plan_bits"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(fn, code):
    if code != TURBO_OK:
        raise TurboError(fn, code)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def params(head_dim=128, block_q=64, block_kv=64, sas_nr=-6, alpha_mode=0, softmax_scale=None, debug_tap=None,
           p_scale_rows=0, scale_fp16=0, sas_fp16=0):
    """turbo_params_t with the paper's defaults.  p_scale_rows=1 selects the
    per-row prefill P scale, scale_fp16=1 the FP16 first-stage scales, sas_fp16=1 the FP16 SAS
    polynomial (NEXT-2 variants, include/turbo_attention.h)."""
    if softmax_scale is None:
        softmax_scale = 1.0 / math.sqrt(head_dim)
    p = TurboParams(head_dim, block_q, block_kv, sas_nr, alpha_mode, softmax_scale, p_scale_rows, scale_fp16,
                    sas_fp16, None)
    if debug_tap is not None:
        p._tap = debug_tap  # keep alive
        p.debug_tap = C.cast(C.pointer(debug_tap.c), C.c_void_p)
    return p


class KVCache:
    """Caller-owned device memory for one layer's compressed cache (torch tensors)."""

    def __init__(self, batch, n_kv_heads, head_dim, max_blocks, bits, block_kv=64, device="cuda"):
        sizes = [C.c_size_t() for _ in range(5)]
        _check("turbo_cache_sizes", lib().turbo_cache_sizes(batch, n_kv_heads, head_dim, block_kv, max_blocks,
                                                            *[C.byref(s) for s in sizes]))
        nrec, npar, nbuf, nau, ncnt = (s.value for s in sizes)
        self.bits = torch.as_tensor(bits, dtype=torch.int32).reshape(n_kv_heads, 2).contiguous()
        self.bits_dev = self.bits.to(device)
        self.block_rec = torch.zeros(max(nrec, 16), dtype=torch.uint8, device=device)
        self.s_parent = torch.zeros(max(npar // 4, 1), dtype=torch.float32, device=device)
        self.buf = torch.zeros(nbuf, dtype=torch.int8, device=device)
        self.a_univ = torch.zeros(nau // 4, dtype=torch.float32, device=device)
        self.counters = torch.zeros(ncnt // 4, dtype=torch.int32, device=device)
        self.c = TurboKVCache(batch, n_kv_heads, head_dim, block_kv, max_blocks, 0, self.bits.data_ptr(),
                              self.bits_dev.data_ptr(), self.block_rec.data_ptr(), self.s_parent.data_ptr(),
                              self.buf.data_ptr(), self.a_univ.data_ptr(), self.counters.data_ptr())
        self.batch, self.n_kv_heads, self.head_dim, self.max_blocks, self.block_kv = (
            batch, n_kv_heads, head_dim, max_blocks, block_kv)

    @property
    def n_tokens(self):
        return self.c.n_tokens

    def rec_bytes(self):
        return 2 * self.head_dim + self.block_kv * self.head_dim // 2

    def records(self):
        """block_rec viewed as [B][Hkv][2][max_blocks][rec_bytes]."""
        return self.block_rec[: self.batch * self.n_kv_heads * 2 * self.max_blocks * self.rec_bytes()].view(
            self.batch, self.n_kv_heads, 2, self.max_blocks, self.rec_bytes())

    def nbytes(self):
        return sum(t.numel() * t.element_size() for t in (self.block_rec, self.s_parent, self.buf, self.a_univ,
                                                          self.counters))


def turbo_quantize_kv(p, cache: KVCache, k, v, mode=0, stream=None, out=None):
    """mode 0 (PREFILL): k, v fp16 [B,N,Hkv,d] -> returns (k1, v1t, k1_scale, v1_scale)
    (written into `out` when given); mode 2 (PREFILL_CHUNK): the same for a further chunk,
    outputs over Nk = cached + N tokens (the chunk at token `cached`; pass `out` holding the
    turbo_dequantize_cache prefix); mode 1 (APPEND): k, v fp16 [B,Hkv,d] -> returns None."""
    assert k.dtype == torch.float16 and v.dtype == torch.float16 and k.is_contiguous() and v.is_contiguous()
    if mode in (0, 2):
        B, N, H, d = k.shape
        Nk = N if mode == 0 else cache.n_tokens + N
        tc = -(-Nk // p.block_kv)
        dev = k.device
        if mode == 2 and out is None:
            # the chunk kernel writes only the chunk's rows; the prefix rows must come from
            # turbo_dequantize_cache (fresh buffers would hand garbage prefix keys on)
            raise ValueError("turbo_quantize_kv mode 2 needs `out` holding the turbo_dequantize_cache prefix")
        if out is not None:
            k1, v1t, k1s, v1s = out
            assert k1.shape == (B, H, Nk, d) and v1t.shape == (B, H, tc, d, p.block_kv)
            assert k1s.shape == (B, H, tc) and v1s.shape == (B, H, tc)
        else:
            k1 = torch.empty((B, H, Nk, d), dtype=torch.float16, device=dev)  # stage-1 codes, exact in fp16
            v1t = torch.empty((B, H, tc, d, p.block_kv), dtype=torch.float16, device=dev)
            k1s = torch.empty((B, H, tc), dtype=torch.float32, device=dev)
            v1s = torch.empty((B, H, tc), dtype=torch.float32, device=dev)
        _check("turbo_quantize_kv", lib().turbo_quantize_kv(C.byref(p), C.byref(cache.c), _ptr(k), _ptr(v), N, mode,
                                                            _ptr(k1), _ptr(v1t), _ptr(k1s), _ptr(v1s),
                                                            _stream(stream)))
        return k1, v1t, k1s, v1s
    _check("turbo_quantize_kv", lib().turbo_quantize_kv(C.byref(p), C.byref(cache.c), _ptr(k), _ptr(v), 1, 1, None,
                                                        None, None, None, _stream(stream)))
    return None


def turbo_attention_prefill(p, q, k1, v1t, k1_scale, v1_scale, causal=True, o=None, lse=None, stream=None):
    """q fp16 [B,N,Hq,d] -> (o fp16 [B,N,Hq,d], lse f32 [B,Hq,N])."""
    assert q.dtype == torch.float16 and q.is_contiguous()
    B, N, Hq, d = q.shape
    Hkv = k1.shape[1]
    if o is None:
        o = torch.empty_like(q)
    if lse is None:
        lse = torch.empty((B, Hq, N), dtype=torch.float32, device=q.device)
    _check("turbo_attention_prefill", lib().turbo_attention_prefill(
        C.byref(p), B, N, Hq, Hkv, int(causal), _ptr(q), _ptr(k1), _ptr(v1t), _ptr(k1_scale), _ptr(v1_scale),
        _ptr(o), _ptr(lse), _stream(stream)))
    return o, lse


def turbo_q_projection(p, x, wq, n_q_heads, want_q16=False, stream=None):
    """Q = x wq^T with the stage-1 Q quantisation fused into the GEMM epilogue:
    x fp16 [B,N,D], wq fp16 [Hq*d, D] -> (q1 int8 [B,N,Hq,d], q1_scale f32 [B,Hq,ceil(N/B_r)],
    q16 fp16 [B,N,Hq,d] or None)."""
    assert x.dtype == torch.float16 and wq.dtype == torch.float16 and x.is_contiguous() and wq.is_contiguous()
    B, N, D = x.shape
    d = p.head_dim
    assert wq.shape == (n_q_heads * d, D)
    dev = x.device
    q1 = torch.empty((B, N, n_q_heads, d), dtype=torch.int8, device=dev)
    sq = torch.empty((B, n_q_heads, -(-N // p.block_q)), dtype=torch.float32, device=dev)
    q16 = torch.empty((B, N, n_q_heads, d), dtype=torch.float16, device=dev) if want_q16 else None
    _check("turbo_q_projection", lib().turbo_q_projection(C.byref(p), B, N, D, n_q_heads, _ptr(x), _ptr(wq), _ptr(q1),
                                                          _ptr(sq), _ptr(q16), _stream(stream)))
    return q1, sq, q16


def turbo_attention_prefill_q1(p, q1, q1_scale, k1, v1t, k1_scale, v1_scale, causal=True, o=None, lse=None,
                               stream=None):
    """Prefill with a pre-quantised query: q1 int8 [B,N,Hq,d], q1_scale [B,Hq,ceil(N/B_r)]
    -> (o fp16 [B,N,Hq,d], lse f32 [B,Hq,N])."""
    assert q1.dtype == torch.int8 and q1.is_contiguous()
    B, N, Hq, d = q1.shape
    Hkv = k1.shape[1]
    if o is None:
        o = torch.empty((B, N, Hq, d), dtype=torch.float16, device=q1.device)
    if lse is None:
        lse = torch.empty((B, Hq, N), dtype=torch.float32, device=q1.device)
    _check("turbo_attention_prefill_q1", lib().turbo_attention_prefill_q1(
        C.byref(p), B, N, Hq, Hkv, int(causal), _ptr(q1), _ptr(q1_scale), _ptr(k1), _ptr(v1t), _ptr(k1_scale),
        _ptr(v1_scale), _ptr(o), _ptr(lse), _stream(stream)))
    return o, lse


def turbo_dequantize_cache(p, cache: KVCache, Nk, blk_begin=0, blk_end=-1, out=None, stream=None):
    """Stage-1 reconstruction of cache blocks [blk_begin, blk_end) into prefill operands over
    Nk tokens -> (k1 fp16 codes [B,Hkv,Nk,d], v1t fp16 [B,Hkv,Tk,d,B_c], k1_scale, v1_scale [B,Hkv,Tk])."""
    B, H, d = cache.batch, cache.n_kv_heads, cache.head_dim
    tk = -(-Nk // p.block_kv)
    if out is None:
        dev = cache.counters.device
        out = (torch.zeros((B, H, Nk, d), dtype=torch.float16, device=dev),
               torch.zeros((B, H, tk, d, p.block_kv), dtype=torch.float16, device=dev),
               torch.zeros((B, H, tk), dtype=torch.float32, device=dev),
               torch.zeros((B, H, tk), dtype=torch.float32, device=dev))
    k1, v1t, k1s, v1s = out
    _check("turbo_dequantize_cache", lib().turbo_dequantize_cache(
        C.byref(p), C.byref(cache.c), blk_begin, blk_end, _ptr(k1), _ptr(v1t), _ptr(k1s), _ptr(v1s), Nk,
        _stream(stream)))
    return out


def turbo_attention_prefill_chunk(p, q, k1, v1t, k1_scale, v1_scale, causal=True, o=None, lse=None, stream=None):
    """Chunked prefill: q fp16 [B,Nq,Hq,d] at positions [Nk-Nq, Nk) against k1 [B,Hkv,Nk,d]
    -> (o fp16 [B,Nq,Hq,d], lse f32 [B,Hq,Nq])."""
    assert q.dtype == torch.float16 and q.is_contiguous()
    B, Nq, Hq, d = q.shape
    Hkv, Nk = k1.shape[1], k1.shape[2]
    if o is None:
        o = torch.empty_like(q)
    if lse is None:
        lse = torch.empty((B, Hq, Nq), dtype=torch.float32, device=q.device)
    _check("turbo_attention_prefill_chunk", lib().turbo_attention_prefill_chunk(
        C.byref(p), B, Nq, Nk, Hq, Hkv, int(causal), _ptr(q), _ptr(k1), _ptr(v1t), _ptr(k1_scale),
        _ptr(v1_scale), _ptr(o), _ptr(lse), _stream(stream)))
    return o, lse


def turbo_decode_workspace_bytes(B, Hq, Hkv, head_dim, n_splits):
    return lib().turbo_decode_workspace_bytes(B, Hq, Hkv, head_dim, n_splits)


def turbo_decode_workers(Hq, Hkv, head_dim):
    return lib().turbo_decode_workers(Hq, Hkv, head_dim)


def balanced_ranges(unit_counts, Hkv, workers, min_units=8):
    """The balanced decode schedule's sub-ranges (include/turbo_attention.h):
    unit_counts[b] = units of each (b, kv head) (blocks + 1 if the buffer block
    is used).  Returns {(b, kvh): [(u0, u1), ...]} in ascending order."""
    total = sum(unit_counts) * Hkv
    C = max(min_units, -(-total // max(1, workers)))
    out, base = {}, 0
    for b, U in enumerate(unit_counts):
        for h in range(Hkv):
            s0, s1 = base, base + U
            out[(b, h)] = [(max(s0, w * C) - s0, min(s1, (w + 1) * C) - s0)
                           for w in range(s0 // C, (s1 - 1) // C + 1)] if U else []
            base = s1
    return out


B200_SMS = 148


def decode_row_groups(G):
    """Row groups per KV head in the decode (include/turbo_attention.h): the least r with G / r <= 8
    query rows that divides G; the schedule then sees Hkv * r (virtual) KV heads of G / r rows."""
    return next(r for r in range(-(-G // 8), G + 1) if G % r == 0)


def reference_workers(Hq, Hkv, head_dim):
    """Resident decode warps of ONE B200 (148 SMs x the decode kernel's warps per SM: 12 for the
    packed G <= 4 path at d = 128, 16 at d = 64, 12 for the general d = 64 path, 8 for the general
    d = 128 path at 250 registers).  The default
    decode schedule uses this fixed count on every device, so that its split partition -- and hence
    its numbers (turbo_attention.h, SPLIT DEPENDENCE) -- never depend on the GPU it runs on; on a
    B200 it equals turbo_decode_workers() (tests/test_gpu_parity.py checks it)."""
    Gv = Hq // Hkv // decode_row_groups(Hq // Hkv)  # rows per (virtual) KV head
    if head_dim == 64:
        per_sm = 16 if Gv <= 4 else 12  # 128 / 165 registers
    else:
        per_sm = 12 if Gv <= 4 else 8   # 168 / 250 registers
    return B200_SMS * per_sm


def auto_splits(batch, n_kv_heads, n_blocks, workers=None):
    """Equal-split count for turbo_attention_decode.  Among the counts that keep >= 8
    blocks per split and whose last split is not short (>= 3/4 of the others, so no
    (b, kv head) ends with a straggler), pick the one whose task count
    batch * n_kv_heads * S is closest to 4.5 waves of the resident decode warps
    (`workers`, default turbo_decode_workers for G <= 4, d = 128).  On B200 this is
    the best of a sweep on configs[2] (S = 12) and within 0.1 % on configs[4] (S = 64;
    tools/sweep_decode.py).  At most 128 splits: the LSE combine runs one CTA per output row, and
    few rows with hundreds of parts each serialise it (B = 1 x 128k: S = 256 39 us, S = 128 35.5 us;
    profiles/r2_small_batch_decode.txt)."""
    if workers is None:
        workers = reference_workers(4, 1, 128)
    bh = max(1, batch * n_kv_heads)
    best, best_err = 1, None
    for s in range(1, min(128, max(1, n_blocks // 8)) + 1):
        per = -(-n_blocks // s)
        last = n_blocks - per * (s - 1)
        if s > 1 and (last <= 0 or 4 * last < 3 * per):
            continue
        err = abs(bh * s / workers - 4.5)
        if best_err is None or err < best_err - 1e-9:
            best, best_err = s, err
    return best


def resolve_splits(n_splits, B, Hq, cache, blk_begin=0, blk_end=-1):
    """The n_splits value turbo_attention_decode passes to the library for a binding-level
    n_splits (None: the deterministic default)."""
    if n_splits is not None:
        return n_splits
    Hkv, d = cache.n_kv_heads, cache.head_dim
    if Hq // Hkv > 4:
        return -reference_workers(Hq, Hkv, d)
    nb = (cache.n_tokens // cache.block_kv) if blk_end < 0 else blk_end
    return auto_splits(B, Hkv, max(0, nb - blk_begin), reference_workers(Hq, Hkv, d))


def turbo_attention_decode(p, cache: KVCache, q, blk_begin=0, blk_end=-1, with_buffer=True, n_splits=1,
                           workspace=None, o=None, o_part=None, lse=None, want_fp16=True, want_f32=False,
                           stream=None):
    """q fp16 [B,Hq,d] -> (o fp16 [B,Hq,d] or None, o_part f32 [B,Hq,d] or None, lse f32 [B,Hq]).
    n_splits >= 1: equal splits; 0: the balanced schedule over this device's workers; -W: the
    balanced schedule over W workers; None (deterministic default, device-independent):
    auto_splits() with reference_workers() for G <= 4, the balanced schedule over
    reference_workers() for G > 4 (the general-path decode is issue-bound: measured 5-10 % faster
    than auto_splits' count on B200 for 8 x 32k, 16 x 32k and 64 x 8k at 64 / 8 heads).  The result
    depends on the partition (turbo_attention.h, SPLIT DEPENDENCE); n_splits = 1 is unsplit Alg. 2."""
    assert q.dtype == torch.float16 and q.is_contiguous()
    B, Hq, d = q.shape
    n_splits = resolve_splits(n_splits, B, Hq, cache, blk_begin, blk_end)
    dev = q.device
    if want_fp16 and o is None:
        o = torch.empty((B, Hq, d), dtype=torch.float16, device=dev)
    if want_f32 and o_part is None:
        o_part = torch.empty((B, Hq, d), dtype=torch.float32, device=dev)
    if lse is None:
        lse = torch.empty((B, Hq), dtype=torch.float32, device=dev)
    wsb = turbo_decode_workspace_bytes(B, Hq, cache.n_kv_heads, d, n_splits)
    if wsb and workspace is None:
        workspace = torch.empty(wsb, dtype=torch.uint8, device=dev)
    _check("turbo_attention_decode", lib().turbo_attention_decode(
        C.byref(p), C.byref(cache.c), Hq, _ptr(q), blk_begin, blk_end, int(with_buffer), n_splits, _ptr(workspace),
        wsb, _ptr(o), _ptr(o_part), _ptr(lse), _stream(stream)))
    return o, o_part, lse


def turbo_combine_lse(o_parts, lse_parts, o=None, o_f32=None, want_fp16=True, stream=None):
    """o_parts f32 [S, rows, d], lse_parts f32 [S, rows] -> (o fp16 | None, o_f32 | None, lse [rows])."""
    S, rows, d = o_parts.shape
    if want_fp16 and o is None:
        o = torch.empty((rows, d), dtype=torch.float16, device=o_parts.device)
    lse = torch.empty((rows,), dtype=torch.float32, device=o_parts.device)
    _check("turbo_combine_lse", lib().turbo_combine_lse(S, rows, d, _ptr(o_parts), _ptr(lse_parts), _ptr(o),
                                                        _ptr(o_f32), _ptr(lse), _stream(stream)))
    return o, o_f32, lse


class DebugTap:
    """Device buffers of a turbo_debug_tap_t (exact-set intermediates of one tile)."""

    def __init__(self, batch, head, i_block, j_block, head_dim, decode=False, device="cuda", block_kv=64):
        rows = 1 if decode else 64
        z = lambda *s, dt: torch.zeros(s, dtype=dt, device=device)  # noqa: E731
        self.q1 = z(rows, head_dim, dt=torch.int8)
        self.s_q = z(1, dt=torch.float32)
        self.s_int = z(rows, block_kv, dt=torch.int32)
        self.m_new = z(rows, dt=torch.float32)
        self.p_codes = z(rows, block_kv, dt=torch.uint8)
        self.s_p = z(1, dt=torch.float32)
        self.pv_int = z(rows, head_dim, dt=torch.int32)
        self.c = TurboDebugTap(batch, head, i_block, j_block, *[t.data_ptr() for t in (
            self.q1, self.s_q, self.s_int, self.m_new, self.p_codes, self.s_p, self.pv_int)])


def turbo_head_priority(k, v, stream=None):
    """Per (kv_head, K/V) slot priority over the prefill K, V fp16 [B,N,Hkv,d]
     -> f64 tensor [Hkv, 2] on the device."""
    assert k.dtype == torch.float16 and k.is_contiguous() and v.is_contiguous()
    B, N, H, d = k.shape
    ws = torch.empty(lib().turbo_priority_workspace_bytes(H, d), dtype=torch.uint8, device=k.device)
    pr = torch.empty((H, 2), dtype=torch.float64, device=k.device)
    _check("turbo_head_priority", lib().turbo_head_priority(B, N, H, d, _ptr(k), _ptr(v), _ptr(ws), ws.numel(),
                                                            _ptr(pr), _stream(stream)))
    return pr


def turbo_plan_bits(priority, n_2bit):
    """Host ranking: the n_2bit lowest-priority slots get 2 bits.
    priority: [Hkv, 2] (any device) -> int32 [Hkv, 2] host tensor."""
    pr = priority.detach().to("cpu", torch.float64).contiguous()
    bits = torch.empty(pr.shape, dtype=torch.int32)
    _check("turbo_plan_bits", lib().turbo_plan_bits(_ptr(pr), pr.numel(), n_2bit, _ptr(bits)))
    return bits


def turbo_selftest_div(which, lo_bits, hi_bits):
    """Exhaustive check of the library's fast correctly rounded divisions
    (which 0: a / 119, 1: 119 / a) against IEEE division over the binary32 bit
    patterns [lo_bits, hi_bits]; returns (mismatches, first mismatching bits)."""
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    first = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    _check("turbo_selftest_div", lib().turbo_selftest_div(which, lo_bits, hi_bits, _ptr(bad), _ptr(first), _stream()))
    torch.cuda.synchronize()
    return int(bad.item()), int(first.item()) & 0xFFFFFFFF
