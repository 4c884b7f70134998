python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k decode > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
SPL3=0,12 SPL5=0,32 timeout 300 python tools/sweep_decode.py
bash tools/ab.sh tools/time_prefill.py variants/pfold.so variants/pfbias.so
TURBO_LIB=variants/profb.so timeout 300 python tools/prof_prefill.py
TURBO_LIB=variants/prof.so timeout 300 python tools/prof_prefill.py
