#!/bin/bash
# A/B of decode variant libraries on the G = 8 (general-path) shapes and configs[2] / [4]: tools/gpu_ab_g8.sh lib1 lib2 ...
python __graft_entry__.py build > /dev/null 2>&1
for rep in 1 2; do for lib in "$@"; do
  echo "== $lib"
  TURBO_LIB=$lib DEC_SHAPES="16,32768,64,8,128;8,32768,64,8,128;1,131072,64,8,128" SPLX=0 timeout 600 python tools/sweep_decode.py
  TURBO_LIB=$lib SPL3=12 SPL5=64 timeout 600 python tools/sweep_decode.py
done; done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
