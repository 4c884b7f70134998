#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chunked.py tests/test_gpu_fullsize.py -q -k "quantize or append or chunk or decode" 2>&1 | tail -2
bash tools/ab.sh tools/time_quant.py variants/comb2.so variants/qsplit.so
