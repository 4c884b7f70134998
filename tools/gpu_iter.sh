#!/bin/bash
# One GPU iteration: prefill parity (+ edge cases) of the in-tree sources, then interleaved timings
# of the given variant libraries (scratch builds under variants/, see tools/README.md).
# Usage: bash tools/gpu_iter.sh <tag> variants/a.so variants/b.so ...   [TP_SHAPE etc. pass through]
tag=${1:-it}; shift
out=gpurun_out/$tag
mkdir -p $out
python __graft_entry__.py build > $out/build.log 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv > $out/clk.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_chunked.py -x -q \
  -k "prefill or tap or zero or clamp or sas or chunk" > $out/pytest.log 2>&1
tail -3 $out/pytest.log
for rep in 1 2 3; do
  for lib in "$@"; do
    TURBO_LIB=$lib timeout 300 python tools/time_prefill.py >> $out/ab.txt 2>&1
  done
done
cat $out/ab.txt
