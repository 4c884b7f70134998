python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "decode or combine or seq" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
export SPL3=8,12 SPL5=32
bash tools/ab_decode.sh variants/d6.so variants/d7.so variants/d6.so variants/d7.so
