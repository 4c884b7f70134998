python __graft_entry__.py build > gpurun_out/build.log 2>&1
SPL3=6,8,9,10,11,12,13,14,15 SPL5=16,20,24,28,30,32,34,36,40 timeout 600 python tools/sweep_decode.py > gpurun_out/sweep.log 2>&1
cat gpurun_out/sweep.log
