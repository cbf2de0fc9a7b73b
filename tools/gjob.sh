L=$PWD/paper_1210_0084_b200
for v in "" nosplit slots8 "" nosplit; do if [ -n "$v" ]; then export SLICQ_LIB=$L/libslicq_$v.so; else unset SLICQ_LIB; fi; echo "== $v"; timeout 300 python tools/e2e_probe.py 32,64 2>&1 | tail -2; done
unset SLICQ_LIB
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "process_host" 2>&1 | tail -2
