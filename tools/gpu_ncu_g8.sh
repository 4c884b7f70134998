#!/bin/bash
# ncu source-level capture of the G = 8 decode (general IMMA path): per-line instruction and stall counts
python __graft_entry__.py build > /dev/null 2>&1
DEC_SHAPE=16,32768,64,8,128 timeout 900 ncu --set full --import-source on --clock-control none -k regex:^decode_kernel -s 1 -c 1 -o gpurun_out/g8 python tools/run_decode.py 0 2 > /dev/null 2>&1
ncu -i gpurun_out/g8.ncu-rep --page source --csv --print-source sass > gpurun_out/g8_source.csv 2>/dev/null
ncu -i gpurun_out/g8.ncu-rep --page raw --csv > gpurun_out/g8_raw.csv 2>/dev/null
rm -f gpurun_out/g8.ncu-rep
ls -la gpurun_out | grep g8
