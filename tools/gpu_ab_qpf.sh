#!/bin/bash
# prefill: L2 prefetch of the next wave's Q rows (TURBO_PREFILL_QPF quarter waves ahead; 0 = off) + prefill GPU tests
python __graft_entry__.py build > /dev/null 2>&1
for rep in 1 2 3; do for q in 0 4 8 2; do
  echo "QPF=$q $(TURBO_PREFILL_QPF=$q python tools/time_prefill.py | tail -1)"
done; done
for q in 0 4; do echo "70b QPF=$q $(TP_CFG=70b TURBO_PREFILL_QPF=$q python tools/time_prefill.py | tail -1)"; done
timeout 1200 python -m pytest tests -m gpu -q -x -k "prefill or chunk or projection or edge" 2>&1 | tail -1
