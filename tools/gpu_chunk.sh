python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_chunked.py -q -x 2>&1 | tail -25
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
bash tools/ab.sh tools/time_prefill.py variants/head.so paper_2412_08585_b200/libturboattn.so
