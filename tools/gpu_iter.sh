#!/bin/bash
# One GPU iteration: prefill parity (+ edge cases) and an A/B of the prefill kernel
# against the round-1 build (variants/v1.so).  Usage: bash tools/gpu_iter.sh <tag>
tag=${1:-it}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv > $out/clk.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_chunked.py -x -q \
  -k "prefill or tap or zero or clamp or sas or chunk" > $out/pytest.log 2>&1
tail -3 $out/pytest.log
for rep in 1 2; do
  for lib in variants/v1.so paper_2412_08585_b200/libturboattn.so; do
    TURBO_LIB=$lib timeout 300 python tools/time_prefill.py >> $out/ab.txt 2>&1
  done
done
cat $out/ab.txt
