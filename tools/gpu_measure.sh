#!/bin/bash
# Full measurement set for one build, tagged: bench lines (all workloads + the reference arm), the ncu launch
# list of the default bench command, `ncu --set full` captures of the three main kernels, the GPU test suite
# and smoke().  Usage: bash tools/gpu_measure.sh <tag> [--no-tests]   (outputs in gpurun_out/<tag>_*)
tag=${1:?tag}
o=gpurun_out/$tag
python __graft_entry__.py build > ${o}_build.log 2>&1
timeout 300 python bench.py > ${o}_bench.json 2>${o}_bench.err
timeout 300 python bench.py --workload decode_long > ${o}_bench_decode_long.json 2>>${o}_bench.err
timeout 600 python bench.py --workload prefill_70b > ${o}_bench_prefill_70b.json 2>>${o}_bench.err
timeout 300 python bench.py --workload prefill_chunk > ${o}_bench_prefill_chunk.json 2>>${o}_bench.err
timeout 300 python bench.py --workload q_projection > ${o}_bench_q_projection.json 2>>${o}_bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > ${o}_bench_reference.json 2>>${o}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file ${o}_launches.csv \
  python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
NCU="ncu --set full --import-source on --clock-control none"
timeout 900 $NCU -k regex:^prefill_kernel -c 1 -o ${o}_prefill python tools/time_prefill.py > /dev/null 2>&1
timeout 900 $NCU -k regex:^decode_kernel -s 1 -c 1 -o ${o}_decode python tools/run_decode.py 12 2 > /dev/null 2>&1
timeout 900 $NCU -k regex:^quant_prefill -c 2 -o ${o}_quant python tools/time_prefill.py > /dev/null 2>&1
# the reports themselves can exceed gpurun's 64 MiB copy-back: keep the summary and the raw pages only
python tools/ncu_summary.py ${o}_launches.csv ${o}_prefill.ncu-rep ${o}_decode.ncu-rep ${o}_quant.ncu-rep \
  > ${o}_ncu_summary.txt 2>&1
for r in prefill decode quant; do
  ncu -i ${o}_$r.ncu-rep --page raw --csv > ${o}_${r}_raw.csv 2>/dev/null
  ncu -i ${o}_$r.ncu-rep --page source --csv > ${o}_${r}_source.csv 2>/dev/null
  rm -f ${o}_$r.ncu-rep
done
if [ "$2" != "--no-tests" ]; then
  timeout 1800 python -m pytest tests -m gpu -q > ${o}_pytest_gpu.log 2>&1
  python __graft_entry__.py smoke > ${o}_smoke.log 2>&1
fi
ls gpurun_out | grep "^$tag"; tail -2 ${o}_pytest_gpu.log 2>/dev/null; tail -1 ${o}_smoke.log 2>/dev/null
