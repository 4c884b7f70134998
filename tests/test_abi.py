"""C-ABI library checks that need no GPU (-m "not gpu"): the shared library
loads, exports every symbol include/turbo_attention.h declares, and its
host-side validation rejects bad arguments before touching the device."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2412_08585_b200 import binding, build

    build.build()
    return binding.lib()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "turbo_attention.h")).read()
    return sorted(set(re.findall(r"^\s*(?:TURBO_API\s+)?(?:const char\*|turbo_status_t|size_t|int32_t)\s+(turbo_\w+)\(", src, re.M)))


def test_header_declares_the_boundary():
    syms = header_symbols()
    for s in ("turbo_quantize_kv", "turbo_attention_prefill", "turbo_attention_decode", "turbo_combine_lse",
              "turbo_decode_workspace_bytes", "turbo_cache_sizes", "turbo_version"):
        assert s in syms


def test_library_exports_every_header_symbol(L):
    from paper_2412_08585_b200 import binding

    for s in header_symbols():
        assert hasattr(L, s), s
    assert set(header_symbols()) == set(binding.EXPORTS)
    assert b"sm_100a" in L.turbo_version()


def test_cache_sizes(L):
    from paper_2412_08585_b200 import binding

    out = [C.c_size_t() for _ in range(5)]
    assert L.turbo_cache_sizes(64, 10, 128, 64, 513, *[C.byref(o) for o in out]) == 0
    rec, par, buf, au, cnt = (o.value for o in out)
    assert rec == 64 * 10 * 2 * 513 * (2 * 128 + 64 * 128 // 2)
    assert par == 64 * 10 * 2 * 513 * 4 and buf == 64 * 10 * 2 * 64 * 128 and au == 64 * 10 * 2 * 4
    assert cnt == 64 * 2 * 4
    assert L.turbo_cache_sizes(1, 1, 96, 64, 1, *[C.byref(o) for o in out]) == binding.TURBO_ERR_UNSUPPORTED
    assert L.turbo_cache_sizes(0, 1, 64, 64, 1, *[C.byref(o) for o in out]) == binding.TURBO_ERR_INVALID_ARG


def test_host_validation_without_gpu(L):
    from paper_2412_08585_b200 import binding as b

    p = b.params(head_dim=128)
    # null / bad arguments are rejected before any CUDA call
    assert L.turbo_attention_prefill(C.byref(p), 1, 64, 3, 2, 1, *[None] * 7, None) == b.TURBO_ERR_UNSUPPORTED
    assert L.turbo_attention_prefill(C.byref(p), 1, 64, 2, 2, 1, *[None] * 7, None) == b.TURBO_ERR_INVALID_ARG
    assert L.turbo_attention_prefill(None, 1, 64, 2, 2, 1, *[None] * 7, None) == b.TURBO_ERR_INVALID_ARG
    bad = b.params(head_dim=128, block_kv=96)  # B_c in {64, 128}
    assert L.turbo_attention_prefill(C.byref(bad), 1, 64, 2, 2, 1, *[None] * 7, None) == b.TURBO_ERR_UNSUPPORTED
    ok128 = b.params(head_dim=128, block_kv=128)
    assert L.turbo_attention_prefill(C.byref(ok128), 1, 64, 2, 2, 1, *[None] * 7, None) == b.TURBO_ERR_INVALID_ARG
    sz = C.c_size_t()
    assert L.turbo_cache_sizes(1, 1, 128, 128, 3, C.byref(sz), None, None, None, None) == b.TURBO_OK
    assert sz.value == 2 * 3 * (2 * 128 + 128 * 128 // 2)
    assert L.turbo_cache_sizes(1, 1, 128, 32, 3, C.byref(sz), None, None, None, None) == b.TURBO_ERR_UNSUPPORTED
    bad = b.params(head_dim=128, sas_nr=0)
    assert L.turbo_attention_prefill(C.byref(bad), 1, 64, 2, 2, 1, *[None] * 7, None) == b.TURBO_ERR_UNSUPPORTED
    assert L.turbo_combine_lse(0, 1, 1, None, None, None, None, None, None) == b.TURBO_ERR_INVALID_ARG
    assert L.turbo_combine_lse(12001, 1, 128, 1, 1, 1, None, 1, None) == b.TURBO_ERR_INVALID_ARG
    # chunked prefill: Nk < Nq, and null operands
    dummy = C.c_void_p(16)
    assert L.turbo_attention_prefill_chunk(C.byref(p), 1, 128, 64, 2, 2, 1, *[dummy] * 7,
                                           None) == b.TURBO_ERR_INVALID_ARG
    assert L.turbo_attention_prefill_chunk(C.byref(p), 1, 64, 128, 2, 2, 1, *[None] * 7,
                                           None) == b.TURBO_ERR_INVALID_ARG
    assert L.turbo_decode_workspace_bytes(2, 8, 2, 128, 1) == 0
    assert L.turbo_decode_workspace_bytes(2, 8, 2, 128, 4) == 4 * 2 * 8 * 129 * 4
    assert L.turbo_decode_workspace_bytes(2, 8, 3, 128, 4) == 0  # Hq % Hkv != 0
    # balanced schedule over an explicit worker count W = -n_splits: (B Hkv + W) G (d + 1) floats
    assert L.turbo_decode_workspace_bytes(2, 8, 2, 128, -1) == (2 * 2 + 1) * 4 * 129 * 4
    assert L.turbo_decode_workspace_bytes(2, 8, 2, 128, -1776) == (2 * 2 + 1776) * 4 * 129 * 4
    assert L.turbo_decode_workspace_bytes(2, 8, 2, 128, -12001) == 0
    assert L.turbo_decode_workspace_bytes(2, 8, 2, 128, 12001) == 0  # n_splits bound (combine weights in smem)
    assert L.turbo_decode_workers(8, 3, 128) == 0
    # quantize_kv / decode with a malformed cache struct
    cache = b.TurboKVCache()
    assert L.turbo_quantize_kv(C.byref(p), C.byref(cache), None, None, 1, 0, None, None, None, None,
                               None) == b.TURBO_ERR_INVALID_ARG
    assert L.turbo_attention_decode(C.byref(p), C.byref(cache), 8, None, 0, -1, 1, 1, None, 0, None, None, None,
                                    None) == b.TURBO_ERR_INVALID_ARG
    assert L.turbo_dequantize_cache(C.byref(p), C.byref(cache), 0, -1, None, None, None, None, 64,
                                    None) == b.TURBO_ERR_INVALID_ARG
    assert L.turbo_quantize_kv(C.byref(p), C.byref(cache), None, None, 64, 2, None, None, None, None,
                               None) == b.TURBO_ERR_INVALID_ARG


def test_sass_uses_tcgen05_and_tma():
    """The prefill kernel's SASS contains tcgen05 MMA (UTC*MMA), TMEM loads
    (LDTM) and TMA loads (UTMALDG); the decode kernel uses bulk copies."""
    import shutil
    import subprocess

    from paper_2412_08585_b200 import build

    lib = build.build()
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    sass = subprocess.run([tool, "-sass", lib], capture_output=True, text=True).stdout
    assert re.search(r"UTC\w*MMA", sass)
    assert "LDTM" in sass
    assert "UTMALDG" in sass
    assert "UBLKCP" in sass


def test_default_decode_schedule_is_device_independent():
    """binding.resolve_splits (the n_splits=None default) depends only on the problem shape, never on
    the device: equal splits by auto_splits over the B200 reference worker count for G <= 4, the
    balanced schedule over that count (n_splits = -W) for G > 4 (include/turbo_attention.h)."""
    from paper_2412_08585_b200 import binding as b

    class FakeCache:
        n_kv_heads, head_dim, block_kv, n_tokens = 10, 128, 64, 32768

    assert b.reference_workers(40, 10, 128) == 148 * 12
    assert b.reference_workers(64, 8, 128) == 148 * 8
    assert b.resolve_splits(None, 64, 40, FakeCache) == b.auto_splits(64, 10, 512, 148 * 12) == 12
    FakeCache.n_kv_heads = 8
    assert b.resolve_splits(None, 8, 64, FakeCache) == -148 * 8
    assert b.resolve_splits(3, 8, 64, FakeCache) == 3


def test_plan_bits_host_only(L):
    """turbo_plan_bits is a host function: runs without a GPU."""
    import numpy as np

    from paper_2412_08585_b200 import binding as b

    pr = np.array([3.0, 1.0, 1.0, 5.0, 0.5, 7.0], np.float64)
    bits = np.zeros(6, np.int32)
    assert L.turbo_plan_bits(pr.ctypes.data_as(C.c_void_p), 6, 3, bits.ctypes.data_as(C.c_void_p)) == 0
    assert bits.tolist() == [4, 2, 2, 4, 2, 4]
    assert L.turbo_plan_bits(pr.ctypes.data_as(C.c_void_p), 6, 7, bits.ctypes.data_as(C.c_void_p)) == \
        b.TURBO_ERR_INVALID_ARG
