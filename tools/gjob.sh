L=$PWD/paper_1210_0084_b200
for v in "" nosnake "" nosnake; do if [ -n "$v" ]; then export SLICQ_LIB=$L/libslicq_$v.so; else unset SLICQ_LIB; fi; echo "== $v"; timeout 120 python tools/quick_time.py 4 2>&1 | grep "fwd:\|inv:"; done
for v in "" nosnake; do if [ -n "$v" ]; then export SLICQ_LIB=$L/libslicq_$v.so; else unset SLICQ_LIB; fi; echo "== cfg3 $v"; timeout 120 python tools/quick_time.py 3 2>&1 | grep "fwd:\|inv:"; echo "== cfg5 $v"; timeout 120 python tools/quick_time.py 5 2>&1 | grep "fwd:\|inv:"; done
