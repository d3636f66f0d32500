#!/bin/bash
# A/B of compile-time library variants in one GPU session:
#   tools/ab_libs.sh "<command>" lib1 lib2 ...   (lib "main" = the product build)
# runs the command twice per variant, interleaved, printing the variant name before each run.
cmd="$1"; shift
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = main ]; then lib=""; else lib="paper_2601_14476_b200/_lib/var_$v/libpbsa.so"; fi
    echo "== $v rep $rep"
    PBSA_LIB="$lib" bash -c "$cmd"
  done
done
