TURBO_LIB=variants/pers.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill" 2>&1 | tail -2
bash tools/ab.sh tools/time_prefill.py variants/pP2.so variants/pers.so
