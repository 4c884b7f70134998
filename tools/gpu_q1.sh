python __graft_entry__.py build > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "quantize or bc128 or chunk or append" 2>&1 | tail -3
for i in 1 2 3; do python tools/time_quant.py; TP_BC=128 python tools/time_quant.py; done
