#!/bin/bash
# A/B/... timing of several builds of libstkb200.so on one box (development tool):
#   tools/abn.sh "<lib1> <lib2> ..." <rounds> <sweep args...>
LIBS=$1; ROUNDS=$2; shift 2
for r in $(seq 1 $ROUNDS); do
  for L in $LIBS; do
    echo "$(basename $L) r$r $(STKB_LIB_LENIENT=1 STKB_LIB=$L python tools/sweep.py "$@" 2>&1 | grep -o '"gpts": [0-9.]*' | paste -sd' ')"
  done
done
