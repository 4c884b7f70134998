#!/bin/bash
# small-batch long-context decode: parity of the in-tree build, split sweep, per-kernel times
python __graft_entry__.py build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py -x -q -k "decode or append or combine or seq" 2>&1 | tail -1
DEC_SHAPES="1,131072,32,8,128;4,32768,32,8,128;1,131072,64,8,128;16,32768,64,8,128" SPLX=0,64,128,192,256,384,512 timeout 600 python tools/sweep_decode.py
DEC_SHAPES="1,131072,32,8,128" SPLX=256 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_kernel|combine" -c 4 python tools/sweep_decode.py 2>&1 | grep -E "decode_kernel|combine_|gpu__time" | head -12
