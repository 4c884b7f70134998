python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_step.json 2> gpurun_out/bench_step.err; echo rc=$?
tail -3 gpurun_out/bench_step.err
timeout 300 python bench.py --workload decode_long > gpurun_out/bench_dlong.json 2>> gpurun_out/bench_step.err
cat gpurun_out/bench_step.json gpurun_out/bench_dlong.json
