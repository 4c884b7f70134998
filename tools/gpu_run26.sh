TURBO_LIB=variants/qV.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "quantize or append" 2>&1 | tail -2
bash tools/ab.sh tools/time_quant.py variants/head.so variants/qV.so
