#!/bin/bash
# B_c = 128: GPU parity (new tests + the B_c = 64 suites as regression) and timings of
# the prefill (configs[1], configs[3]) and decode (configs[2], configs[4]) at both block sizes.
o=gpurun_out/${1:-bc128}
python __graft_entry__.py build > ${o}_build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > ${o}_pytest.log 2>&1
tail -3 ${o}_pytest.log
for bc in 64 128; do
  TP_BC=$bc timeout 120 python tools/time_prefill.py
  TP_BC=$bc TP_CFG=70b timeout 300 python tools/time_prefill.py
  TP_BC=$bc SPL3=0,8,12 SPL5=0,32,64 timeout 300 python tools/sweep_decode.py
done > ${o}_timing.txt 2>&1
cat ${o}_timing.txt
