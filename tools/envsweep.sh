#!/bin/bash
# Dev tool: cfg4 timing under env / library switches (tools/quick_time.py), 2 rounds
L=$PWD/paper_1210_0084_b200
run() { echo "== $1: $(env $1 python tools/quick_time.py ${CFG:-4} 2>&1 | grep -E '^(fwd|inv)' | awk '{printf "%s %s ms  ", $1, $2}')"; }
for r in 1 2; do
  run "X=0"
  for v in "$@"; do run "$v"; done
done
