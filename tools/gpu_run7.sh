python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
SPL3=0,12,8 SPL5=0,32 timeout 600 python tools/sweep_decode.py > gpurun_out/sweep.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_step.json 2> gpurun_out/bench_step.err
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/sweep.log; cat gpurun_out/bench_step.json
