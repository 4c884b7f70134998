python __graft_entry__.py build > gpurun_out/build.log 2>&1
TURBO_PREFILL_NS1=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k prefill > gpurun_out/pytest_ns1.log 2>&1; echo pytest_ns1=$?; tail -2 gpurun_out/pytest_ns1.log
for i in 1 2; do timeout 300 python tools/time_prefill.py; TURBO_PREFILL_NS1=1 timeout 300 python tools/time_prefill.py; done
NCU="ncu --set full --clock-control none"
timeout 900 $NCU -k regex:decode_kernel -s 1 -c 1 -o gpurun_out/dec_S0 python tools/run_decode.py 0 2 > /dev/null 2>&1
timeout 900 $NCU -k regex:decode_kernel -s 1 -c 1 -o gpurun_out/dec_S12 python tools/run_decode.py 12 2 > /dev/null 2>&1
ls gpurun_out
