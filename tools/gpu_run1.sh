set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python bench.py > gpurun_out/bench_step.json 2> gpurun_out/bench_step.err
timeout 300 python bench.py --workload decode_long > gpurun_out/bench_dlong.json 2>> gpurun_out/bench_step.err
timeout 600 python bench.py --workload prefill_70b > gpurun_out/bench_p70.json 2>> gpurun_out/bench_step.err
timeout 300 python tools/sweep_decode.py > gpurun_out/sweep.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench_*.json
