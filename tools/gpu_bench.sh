python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python bench.py > gpurun_out/bench_step.json 2>gpurun_out/bench.err; echo rc=$?
timeout 300 python bench.py --workload decode_long > gpurun_out/bench_dlong.json 2>>gpurun_out/bench.err; echo rc=$?
tail -2 gpurun_out/bench.err; python -c "
import json; d=json.load(open('gpurun_out/bench_step.json')); print(d['value'], d['roofline']['frac'], d['e2e'], d['decode']['n_splits'], d['decode']['kv_gbs'], d['decode']['roofline']['frac'])
d=json.load(open('gpurun_out/bench_dlong.json')); print(d['value'])"
