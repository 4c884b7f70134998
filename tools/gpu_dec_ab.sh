#!/bin/bash
# decode A/B across libraries: parity of the candidate, then interleaved sweeps
cand=${1:-variants/sft.so}
TURBO_LIB=$cand timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q -k "decode or append or combine or sas_fp16" 2>&1 | tail -1
export DEC_SHAPES="64,32768,40,10,128;16,131072,32,8,128;16,32768,64,8,128" SPLX=0,8,12,32,64
for rep in 1 2; do for lib in variants/r2start.so variants/head.so $cand; do echo "== $lib"; TURBO_LIB=$lib timeout 600 python tools/sweep_decode.py; done; done
