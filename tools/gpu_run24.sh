python __graft_entry__.py build > gpurun_out/build.log 2>&1
numactl -H 2>/dev/null | head -3; nvidia-smi topo -m 2>/dev/null | head -4
python tools/pcie_probe.py
for i in 1 2; do timeout 300 python bench.py --no-decode 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e'])"; done
