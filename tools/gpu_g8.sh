#!/bin/bash
# G = 8 decode A/B: parity of each variant, then a sweep over G = 8 shapes for each library.
for lib in "$@"; do
  echo "== parity $lib"
  TURBO_LIB=$lib timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "decode or seq" 2>&1 | tail -1
done
export DEC_SHAPES="8,32768,64,8,128;64,8192,64,8,128;16,32768,64,8,128;32,16384,32,4,128" SPLX=0,16,32,64
bash tools/ab_decode.sh "$@" "$@"
