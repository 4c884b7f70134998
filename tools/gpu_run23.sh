python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill" 2>&1 | tail -2
bash tools/ab.sh tools/time_prefill.py variants/pP2.so variants/pQ16.so variants/pQ32.so
