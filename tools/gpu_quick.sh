#!/bin/bash
# full GPU test suite + the default bench line (quick check of a build)
python __graft_entry__.py build > gpurun_out/quick_build.log 2>&1 || { tail -20 gpurun_out/quick_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 600 python bench.py > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err; tail -c 600 gpurun_out/quick_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/quick_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], json.dumps(d['roofline']), json.dumps(d.get('deviation',{}).get('variants')))"
