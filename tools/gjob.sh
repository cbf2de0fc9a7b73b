for i in 1 2; do timeout 120 python tools/quick_time.py 5 2>&1 | grep "fwd:\|inv:"; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg5 or range or large or 131072 or other_slice" > gpurun_out/g11_tests.txt 2>&1; tail -3 gpurun_out/g11_tests.txt
