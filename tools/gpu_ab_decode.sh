#!/bin/bash
# decode A/B: parity of each variant, then configs[2] / configs[4] and G = 8 sweeps per library
for lib in "$@"; do
  echo "== parity $lib"
  TURBO_LIB=$lib timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "decode or seq or combine" 2>&1 | tail -1
done
SPL3=0 SPL5=0 bash tools/ab_decode.sh variants/head.so "$@" variants/head.so "$@"
export DEC_SHAPES="8,32768,64,8,128;16,32768,64,8,128;64,8192,64,8,128" SPLX=0,16,32
bash tools/ab_decode.sh variants/head.so "$@" variants/head.so "$@"
