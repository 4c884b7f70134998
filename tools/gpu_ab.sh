# tools/gpu_ab.sh: parity of a variant library + interleaved timing against variants/head.so
# usage: bash tools/gpu_ab.sh <variant.so> <pytest -k expr> <timing script>
TURBO_LIB=$1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "$2" 2>&1 | tail -1
bash tools/ab.sh $3 variants/head.so $1
