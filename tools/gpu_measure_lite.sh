#!/bin/bash
# Measurement set without the ncu --set full captures (they can exceed gpurun's 64 MiB copy-back):
# bench lines of every workload + the reference arm, the ncu launch list, GPU tests, smoke.
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
timeout 1800 python -m pytest tests -m gpu -q > ${o}_pytest_gpu.log 2>&1
python __graft_entry__.py smoke > ${o}_smoke.log 2>&1
ls gpurun_out | grep "^$tag"; tail -2 ${o}_pytest_gpu.log; tail -1 ${o}_smoke.log
