python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_step.json 2>gpurun_out/bench.err; echo rc=$?
tail -2 gpurun_out/bench.err; python -c "import json; d=json.load(open('gpurun_out/bench_step.json')); print(d['value'], d['roofline'], d['e2e']['value'], d['decode']['kv_gbs'])"
