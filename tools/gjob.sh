L=$PWD/paper_1210_0084_b200
for v in "" nopf2 "" nopf2; do if [ -n "$v" ]; then export SLICQ_LIB=$L/libslicq_$v.so; else unset SLICQ_LIB; fi; echo "== $v"; timeout 120 python tools/quick_time.py 4 2>&1 | grep "inv:"; timeout 120 python tools/quick_time.py 3 2>&1 | grep "inv:"; done
