TURBO_LIB=variants/dS.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "decode" 2>&1 | tail -2
export SPL3=8,12 SPL5=32
bash tools/ab_decode.sh variants/head.so variants/dS.so variants/head.so variants/dS.so
