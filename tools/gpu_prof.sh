# ncu --set full (+source) of the prefill and decode kernels; reports land in gpurun_out/
python __graft_entry__.py build > gpurun_out/build.log 2>&1
NCU="ncu --set full --import-source on --clock-control none"
timeout 900 $NCU -k regex:prefill_kernel -c 1 -o gpurun_out/prefill_full python tools/time_prefill.py > gpurun_out/ncu_prefill.log 2>&1
timeout 900 $NCU -k regex:decode_kernel -s 2 -c 1 -o gpurun_out/decode_full python tools/run_decode.py 8 3 > gpurun_out/ncu_decode.log 2>&1
ls -la gpurun_out
