TURBO_LIB=variants/pW.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill" 2>&1 | grep -E "^E |FAILED|Error|test_" | head -30
