python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
export SPL3=8,10,12,16 SPL5=24,32,40
timeout 300 python tools/sweep_decode.py > gpurun_out/sweep.log 2>&1
TURBO_LIB=variants/v1.so SPL3=8,12 SPL5=32 timeout 300 python tools/sweep_decode.py >> gpurun_out/sweep.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/sweep.log
