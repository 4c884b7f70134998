python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 300 python bench.py > gpurun_out/r1v13_bench.json 2>/dev/null
timeout 300 python bench.py --workload decode_long > gpurun_out/r1v13_bench_decode_long.json 2>/dev/null
timeout 600 python bench.py --workload prefill_70b > gpurun_out/r1v13_bench_prefill_70b.json 2>/dev/null
timeout 300 python bench.py --workload prefill_chunk > gpurun_out/r1v13_bench_prefill_chunk.json 2>/dev/null
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1v13_bench_reference.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r1v13_launches.csv python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
NCU="ncu --set full --import-source on --clock-control none"
timeout 900 $NCU -k regex:^prefill_kernel -c 1 -o gpurun_out/r1v13_prefill python tools/time_prefill.py > /dev/null 2>&1
timeout 900 $NCU -k regex:^decode_kernel -s 1 -c 1 -o gpurun_out/r1v13_decode python tools/run_decode.py 12 2 > /dev/null 2>&1
timeout 900 $NCU -k regex:^quant_prefill_kernel -c 2 -o gpurun_out/r1v13_quant python tools/time_prefill.py > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r1v13_pytest_gpu.log 2>&1
python __graft_entry__.py smoke > gpurun_out/r1v13_smoke.log 2>&1
ls gpurun_out | grep r1v13; tail -2 gpurun_out/r1v13_pytest_gpu.log; cat gpurun_out/r1v13_smoke.log | tail -1
