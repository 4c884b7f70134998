python __graft_entry__.py build > gpurun_out/build.log 2>&1
SPL3=8,10,12,14,16,20 SPL5=32,40,48,56,64 timeout 600 python tools/sweep_decode.py
