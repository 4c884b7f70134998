"""Build libturboattn.so (sm_100a only) in-tree with nvcc.

    python -m paper_2412_08585_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libturboattn.so")
SOURCES = ["api.cu", "quantize.cu", "prefill.cu", "decode.cu", "projection.cu", "planner.cu", "selftest.cu"]
HEADERS = ["common.cuh", "layout.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "turbo_attention.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, csrc: str = None, out: str = None) -> str:
    """Compile csrc/*.cu into `out` (default: the in-tree libturboattn.so).
    `csrc`/`out` let tools/ build A/B variants of the sources side by side."""
    if csrc is not None or out is not None:
        return _build(csrc or CSRC, out or LIB, verbose)
    if not force and not _stale():
        return LIB
    return _build(CSRC, LIB, verbose)


def _build(csrc: str, lib: str, verbose: bool) -> str:
    objdir = os.path.join(PKG, "_obj", os.path.basename(lib).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        flags = [f if f != CSRC else csrc for f in FLAGS]
        cmd = [NVCC, *ARCH, *flags, "-c", os.path.join(csrc, src), "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
            print(" ".join(cmd), flush=True)
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if out and (verbose or p.returncode):
            sys.stdout.write(out.decode())
        if p.returncode:
            failed = True
    if failed:
        raise RuntimeError("nvcc failed")
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
