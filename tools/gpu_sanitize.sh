# compute-sanitizer memcheck / racecheck / synccheck over smoke() and small parity cases
python __graft_entry__.py build > gpurun_out/build.log 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/san_memcheck_smoke.log 2>&1; echo memcheck_smoke=$?
timeout 1200 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "decode_parity or combine or quantize_kv_prefill or prefill_parity" > gpurun_out/san_memcheck_tests.log 2>&1; echo memcheck_tests=$?
timeout 900 $CS --tool racecheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/san_racecheck_smoke.log 2>&1; echo racecheck_smoke=$?
timeout 900 $CS --tool synccheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/san_synccheck_smoke.log 2>&1; echo synccheck_smoke=$?
tail -3 gpurun_out/san_*.log
