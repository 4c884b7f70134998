#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chunked.py tests/test_gpu_fullsize.py -q -k "prefill" 2>&1 | tail -2
python __graft_entry__.py smoke 2>&1 | tail -1
for shp in "8,4096,32,8,128" "8,4096,32,32,128" "8,4096,32,8,64"; do
  TP_SHAPE=$shp bash tools/ab.sh tools/time_prefill.py variants/comb2.so variants/smax.so
done
