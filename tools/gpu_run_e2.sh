python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k prefill 2>&1 | tail -1
bash tools/ab.sh tools/time_prefill.py variants/head.so variants/pE2.so
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck python __graft_entry__.py smoke > gpurun_out/san_racecheck_smoke.log 2>&1
grep -h "Race reported between" gpurun_out/san_racecheck_smoke.log | sed 's/+0x[0-9a-f]*//' | sort | uniq -c
tail -2 gpurun_out/san_racecheck_smoke.log
