python __graft_entry__.py build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
export SPL3=8,12 SPL5=32
bash tools/ab_decode.sh variants/head.so variants/dC.so variants/head.so variants/dC.so
