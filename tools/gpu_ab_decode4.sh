#!/bin/bash
# decode A/B of variant libraries on the packed (G <= 4) path: configs[2] / [4] and small batches, 3 reps; GPU tests
python __graft_entry__.py build > /dev/null 2>&1
for rep in 1 2 3; do for lib in "$@"; do
  echo "== $lib"
  TURBO_LIB=$lib SPL3=12 SPL5=64 timeout 600 python tools/sweep_decode.py
  TURBO_LIB=$lib DEC_SHAPES="1,131072,32,8,128;4,32768,32,8,128" SPLX=128,64 timeout 600 python tools/sweep_decode.py
done; done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
