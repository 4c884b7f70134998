#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over smoke() and small parity cases (B200).
# Usage: bash tools/gpu_sanitize.sh [tag]   (logs in gpurun_out/<tag>_san_*.log)
t=${1:-san}
python __graft_entry__.py build > gpurun_out/${t}_build.log 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/${t}_memcheck_smoke.log 2>&1; echo memcheck_smoke=$?
timeout 1500 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bc128.py -x -q -k "decode_parity or combine or quantize_kv or prefill_parity" > gpurun_out/${t}_memcheck_tests.log 2>&1; echo memcheck_tests=$?
timeout 900 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/${t}_racecheck_smoke.log 2>&1; echo racecheck_smoke=$?
timeout 1200 $CS --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "quantize_kv_prefill_bit_exact or decode_parity" > gpurun_out/${t}_racecheck_tests.log 2>&1; echo racecheck_tests=$?
timeout 900 $CS --tool synccheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/${t}_synccheck_smoke.log 2>&1; echo synccheck_smoke=$?
timeout 900 $CS --tool initcheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/${t}_initcheck_smoke.log 2>&1; echo initcheck_smoke=$?
for f in gpurun_out/${t}_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|Race reported|Barrier error|passed|failed|Error" $f | sort | uniq -c | head -12; done
