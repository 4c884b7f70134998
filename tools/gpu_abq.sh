TURBO_LIB=variants/qL3.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "quantize or append" 2>&1 | tail -1
bash tools/ab.sh tools/time_quant.py variants/head.so variants/qL3.so variants/qL4.so
