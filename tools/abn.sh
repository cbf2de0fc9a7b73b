#!/bin/bash
# Dev tool: timing of several library builds (tools/quick_time.py, alternating, 2 rounds)
# usage: tools/abn.sh "4 3" libA.so libB.so ...
CFGS=$1; shift
for r in 1 2; do
  for c in $CFGS; do
    for L in "$@"; do
      echo "== $(basename $L) cfg$c: $(SLICQ_LIB=$L python tools/quick_time.py $c 2>&1 | grep -E '^(fwd|inv)' | awk '{printf "%s %s ms  ", $1, $2}')"
    done
  done
done
