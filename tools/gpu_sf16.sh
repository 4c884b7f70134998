#!/bin/bash
# sas_fp16 variant + integer stage-2 quantiser: GPU tests, timings (prefill both SAS, quantize A/B)
python __graft_entry__.py build > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for rep in 1 2; do
  python tools/time_prefill.py; TP_SF16=1 python tools/time_prefill.py
done
for rep in 1 2 3; do for lib in variants/head.so variants/qv3.so; do TURBO_LIB=$lib timeout 300 python tools/time_quant.py; done; done
