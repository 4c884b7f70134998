TURBO_LIB=variants/dLI.so timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "decode" 2>&1 | tail -2
export SPL3=8,12 SPL5=32
bash tools/ab_decode.sh variants/d6.so variants/dL.so variants/dI.so variants/dLI.so
