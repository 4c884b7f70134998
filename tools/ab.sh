#!/bin/bash
# tools/ab.sh <script> lib1 lib2 ...   (run a timing script against each library, twice, interleaved)
script=$1; shift
for rep in 1 2; do for lib in "$@"; do TURBO_LIB=$lib timeout 300 python $script; done; done
