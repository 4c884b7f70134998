#!/bin/bash
# K^q1 as fp16 codes + kind::f16 QK^T: full GPU suite, then prefill / quantize timings vs the previous build
python __graft_entry__.py build > gpurun_out/k16_build.log 2>&1 || { tail -30 gpurun_out/k16_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
for r in 1 2; do for l in variants/head.so paper_2412_08585_b200/libturboattn.so; do
  TURBO_LIB=$l python tools/time_prefill.py; TURBO_LIB=$l TP_CFG=70b python tools/time_prefill.py; TURBO_LIB=$l TP_BC=128 python tools/time_prefill.py
  TURBO_LIB=$l python tools/time_quant.py; done; done
