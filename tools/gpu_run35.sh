python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
TURBO_LIB=variants/pQc.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill" 2>&1 | tail -1
bash tools/ab.sh tools/time_prefill.py variants/head.so variants/pQc.so
