for i in 1 2; do timeout 120 python tools/quick_time.py 4 2>&1 | grep "fwd:\|inv:"; done
timeout 120 python tools/quick_time.py 3 2>&1 | grep "fwd:\|inv:"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/g6_tests.txt 2>&1; tail -3 gpurun_out/g6_tests.txt
