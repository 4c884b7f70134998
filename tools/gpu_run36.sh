TURBO_LIB=variants/pQd.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill" 2>&1 | tail -1
bash tools/ab.sh tools/time_prefill.py variants/head.so variants/pQd.so
