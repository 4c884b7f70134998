#!/bin/bash
# one ncu --set full capture of quant_prefill_kernel (configs[1]) -> gpurun_out/<tag>_quant_{raw,source}.csv + summary
tag=${1:?tag}
python __graft_entry__.py build > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:^quant_prefill -s 3 -c 1 \
  -o gpurun_out/${tag}_quant python tools/time_quant.py > /dev/null 2>&1
python tools/ncu_summary.py /dev/null gpurun_out/${tag}_quant.ncu-rep > gpurun_out/${tag}_quant_summary.txt 2>&1
ncu -i gpurun_out/${tag}_quant.ncu-rep --page raw --csv > gpurun_out/${tag}_quant_raw.csv 2>/dev/null
ncu -i gpurun_out/${tag}_quant.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_quant_source.csv 2>/dev/null
ncu -i gpurun_out/${tag}_quant.ncu-rep --page details > gpurun_out/${tag}_quant_details.txt 2>/dev/null
rm -f gpurun_out/${tag}_quant.ncu-rep
ls -la gpurun_out | grep ${tag}_quant
