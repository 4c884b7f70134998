python __graft_entry__.py build > gpurun_out/build.log 2>&1
for sg in 0 100 250 500; do echo stagger=$sg; TURBO_DECODE_STAGGER=$sg SPL3=0 SPL5=0 timeout 300 python tools/sweep_decode.py; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dec_launches_S0.csv python tools/run_decode.py 0 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dec_launches_S12.csv python tools/run_decode.py 12 3 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/dec_launches_S0.csv; python tools/ncu_summary.py gpurun_out/dec_launches_S12.csv
