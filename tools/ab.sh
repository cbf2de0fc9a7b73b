#!/bin/bash
# Dev tool: A/B timing of two library builds (tools/quick_time.py, alternating, 2 rounds)
# usage: tools/ab.sh libA.so libB.so "4 3 5"
A=$1; B=$2; CFGS=${3:-"4 3 5"}
for r in 1 2; do
  for c in $CFGS; do
    for L in $A $B; do
      echo "== $(basename $L) cfg$c: $(SLICQ_LIB=$L python tools/quick_time.py $c 2>&1 | grep -E '^(fwd|inv)' | awk '{printf "%s %s ms  ", $1, $2}')"
    done
  done
done
