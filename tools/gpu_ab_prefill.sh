#!/bin/bash
# prefill A/B: GPU prefill parity of the candidate, then interleaved timings against variants/head.so
cand=${1:?candidate .so}
TURBO_LIB=$cand timeout 900 python -m pytest tests -m gpu -q -x -k "prefill or bc128 or chunk or projection or sas_fp16 or edge" 2>&1 | tail -2
for r in 1 2 3; do for l in variants/head.so $cand; do TURBO_LIB=$l python tools/time_prefill.py; done; done
for l in variants/head.so $cand; do TURBO_LIB=$l TP_BQ=128 python tools/time_prefill.py; TURBO_LIB=$l TP_CFG=70b python tools/time_prefill.py; done
