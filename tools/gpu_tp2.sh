#!/bin/bash
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chunked.py tests/test_gpu_fullsize.py -q -k "prefill" 2>&1 | tail -30
