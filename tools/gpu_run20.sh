timeout 300 python bench.py > gpurun_out/bench_step.json 2> gpurun_out/bench_step.err; echo rc=$?
tail -3 gpurun_out/bench_step.err
cat gpurun_out/bench_step.json
bash tools/ab.sh tools/time_prefill.py variants/pP0.so variants/pP2.so
