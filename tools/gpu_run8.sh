python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for W in 0 7680 3552 5328; do echo W=$W; TURBO_DECODE_WORKERS=$W SPL3=0 SPL5=0 timeout 300 python tools/sweep_decode.py; done
bash tools/ab.sh tools/time_prefill.py variants/v1.so variants/v3.so
