TURBO_LIB=$1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "decode or combine or seq" 2>&1 | tail -1
export SPL3=8,12,16 SPL5=32,64
bash tools/ab_decode.sh variants/head.so $1 variants/head.so $1
