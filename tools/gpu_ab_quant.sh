#!/bin/bash
# quantize_kv A/B over variant libraries (TMA persistent kernel variants) + the in-tree build's GPU tests
python __graft_entry__.py build > /dev/null 2>&1
for i in 1 2; do for lib in "$@"; do
  for bc in 64 128; do echo "BC=$bc $(TP_BC=$bc TURBO_LIB=$lib python tools/time_quant.py 2>&1 | tail -1)"; done
done; done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
