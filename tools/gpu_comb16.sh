#!/bin/bash
TURBO_LIB=variants/c16.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q -k "decode or append or combine" 2>&1 | tail -1
export DEC_SHAPES="1,131072,32,8,128;4,32768,32,8,128;64,32768,40,10,128;16,131072,32,8,128" SPLX=0,64,128,256
for rep in 1 2; do for lib in variants/head.so variants/c16.so; do echo "== $lib"; TURBO_LIB=$lib timeout 600 python tools/sweep_decode.py; done; done
