#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "decode or seq or combine" 2>&1 | tail -1
SPL3=0,12 SPL5=0,64 bash tools/ab_decode.sh variants/head.so variants/comb.so variants/comb2.so
export DEC_SHAPES="1,131072,32,8,128;4,32768,32,8,128;8,32768,64,8,128" SPLX=0,128,256
bash tools/ab_decode.sh variants/head.so variants/comb.so variants/comb2.so
