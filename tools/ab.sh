#!/bin/bash
# A/B timing of two builds of libstkb200.so on the same box (development tool):
#   tools/ab.sh <libA> <libB> <sweep args...>   (alternates A B A B, 2 rounds)
A=$1; B=$2; shift 2
for r in 1 2; do
  for L in $A $B; do
    echo "== $(basename $L) round $r"
    STKB_LIB_LENIENT=1 STKB_LIB=$L python tools/sweep.py "$@" 2>&1 | grep gpts
  done
done
