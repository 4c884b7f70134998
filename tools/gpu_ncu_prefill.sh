#!/bin/bash
# one ncu --set full capture of the prefill kernel (and its summary) -> gpurun_out/<tag>_prefill.*
tag=${1:?tag}
python __graft_entry__.py build > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:^prefill_kernel -c 1 -o gpurun_out/${tag}_prefill python tools/time_prefill.py > /dev/null 2>&1
python tools/ncu_summary.py /dev/null gpurun_out/${tag}_prefill.ncu-rep > gpurun_out/${tag}_prefill_summary.txt 2>&1
ncu -i gpurun_out/${tag}_prefill.ncu-rep --page raw --csv > gpurun_out/${tag}_prefill_raw.csv 2>/dev/null
rm -f gpurun_out/${tag}_prefill.ncu-rep
ls -la gpurun_out | grep $tag
