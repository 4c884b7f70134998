#!/bin/bash
# query-tile pairing for odd G: parity (in-tree build) + prefill timing head vs variant
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chunked.py -x -q -k "prefill" 2>&1 | tail -2
for shp in "8,4096,32,8,128" "8,4096,32,32,128" "8,4096,40,40,128" "4,8192,32,32,128" "8,4096,32,32,64" "16,2048,24,8,128"; do
  TP_SHAPE=$shp bash tools/ab.sh tools/time_prefill.py variants/head.so variants/tp.so
done
