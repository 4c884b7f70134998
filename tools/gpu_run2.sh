export SPL3=8,12 SPL5=24,32
bash tools/ab_decode.sh variants/base.so variants/v1.so > gpurun_out/ab_decode.log 2>&1
bash tools/ab_decode.sh variants/base.so variants/v1.so >> gpurun_out/ab_decode.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:^prefill_kernel -c 1 -o gpurun_out/prefill_full python tools/time_prefill.py > gpurun_out/ncu_prefill.log 2>&1
