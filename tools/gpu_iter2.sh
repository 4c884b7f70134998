#!/bin/bash
# gpu_iter.sh plus the MHA (G = 1), d = 64, N = 1k shapes and the per-row P scale / B_r = 128 variants.
# Usage: bash tools/gpu_iter2.sh <tag> libs...
tag=$1
bash tools/gpu_iter.sh "$@"
shift
for lib in "$@"; do
  for env in "TP_SHAPE=8,4096,32,32,128" "TP_SHAPE=8,4096,32,8,64" "TP_SHAPE=8,1024,32,8,128" "TP_PROW=1" "TP_BQ=128"; do
    echo -n "$env " >> gpurun_out/$tag/ab.txt
    env $env TURBO_LIB=$lib timeout 300 python tools/time_prefill.py >> gpurun_out/$tag/ab.txt 2>&1
  done
done
tail -12 gpurun_out/$tag/ab.txt
