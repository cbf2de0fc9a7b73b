mkdir -p gpurun_out/m2
python bench.py > gpurun_out/m2/bench_cfg4.json 2> gpurun_out/m2/bench_cfg4.err; tail -1 gpurun_out/m2/bench_cfg4.json | cut -c1-200
for c in 1 2 3 5; do python bench.py --config $c --steps 30 > gpurun_out/m2/bench_cfg$c.json 2> gpurun_out/m2/bench_cfg$c.err; tail -1 gpurun_out/m2/bench_cfg$c.json | cut -c1-120; done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/m2/bench_ref.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/m2/launches_cfg4.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/m2/ncu_launch.log 2>&1
SLICQ_PIPE=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:slicq_ --launch-skip 6 --launch-count 6 -o /tmp/mfull python tools/prof_once.py 4 172800000 1 > gpurun_out/m2/ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/mfull.ncu-rep > gpurun_out/m2/ncu_full_summary.txt 2>&1
python tools/ncu_traffic.py /tmp/mfull.ncu-rep cfg4 gpurun_out/m2/ncu_traffic_cfg4.json > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/m2/gpu_tests.txt 2>&1; tail -2 gpurun_out/m2/gpu_tests.txt
