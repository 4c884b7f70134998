python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
export SPL3=8,12,16 SPL5=24,32,48
bash tools/ab_decode.sh variants/v1.so variants/v2.so variants/v1.so variants/v2.so > gpurun_out/ab_decode.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/ab_decode.log
