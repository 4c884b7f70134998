#!/bin/bash
# quantize_kv A/B: parity of the candidate library, then interleaved timings (tools/time_quant.py)
cand=${1:-variants/qpers.so}
TURBO_LIB=$cand timeout 900 python -m pytest tests -m gpu -x -q -k "quantize or append or bc128 or chunk or planner or fullsize" 2>&1 | tail -2
for rep in 1 2 3; do for lib in variants/head.so $cand; do TURBO_LIB=$lib timeout 300 python tools/time_quant.py; TP_BC=128 TURBO_LIB=$lib timeout 300 python tools/time_quant.py; done; done
