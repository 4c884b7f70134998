#!/bin/bash
# A/B of decode variant libraries on the G = 8 (general-path) shapes: tools/gpu_ab_g8.sh lib1 lib2 ...
for lib in "$@"; do
  echo "== $lib"
  TURBO_LIB=$lib DEC_SHAPES="16,32768,64,8,128;8,32768,64,8,128;64,8192,64,8,128;1,131072,64,8,128" \
    SPLX=0,-1184,-1628 timeout 600 python tools/sweep_decode.py
done
TURBO_LIB=$2 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "decode" 2>&1 | tail -1
