TURBO_LIB=variants/prof.so timeout 300 python tools/prof_prefill.py > gpurun_out/prof_prefill.log 2>&1
cat gpurun_out/prof_prefill.log
