python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1v6_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/r1v6_bench_under_ncu.log 2>&1
NCU="ncu --set full --import-source on --clock-control none"
timeout 900 $NCU -k regex:^prefill_kernel -c 1 -o gpurun_out/r1v6_prefill python tools/time_prefill.py > /dev/null 2>&1
timeout 900 $NCU -k regex:^decode_kernel -s 1 -c 1 -o gpurun_out/r1v6_decode python tools/run_decode.py 8 2 > /dev/null 2>&1
timeout 900 $NCU -k regex:^quant_prefill_kernel -c 1 -o gpurun_out/r1v6_quant python tools/time_prefill.py > /dev/null 2>&1
timeout 300 python bench.py > gpurun_out/r1v6_bench.json 2>/dev/null
ls -la gpurun_out
