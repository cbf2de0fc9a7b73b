for i in 1 2; do timeout 120 python tools/quick_time.py 4 2>&1 | grep "fwd:\|inv:"; done
timeout 120 python tools/quick_time.py 3 2>&1 | grep "fwd:\|inv:"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g7_tests.txt 2>&1; tail -3 gpurun_out/g7_tests.txt
