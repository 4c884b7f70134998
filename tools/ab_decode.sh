#!/bin/bash
# A/B the decode kernel of variant libraries in one box session: tools/ab_decode.sh lib1 lib2 ...
for lib in "$@"; do
  echo "== $lib"
  TURBO_LIB=$lib timeout 600 python tools/sweep_decode.py
done
