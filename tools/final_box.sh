#!/bin/bash
# Dev tool (GPU box): the round's final records -- GPU tests, bench lines of every config, the
# reference arm, the ncu launch list of the bench command and the ncu full summary.
mkdir -p gpurun_out/final
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/final/gpu_tests.log 2>&1
tail -3 gpurun_out/final/gpu_tests.log
python bench.py > gpurun_out/final/bench_r2.json 2> gpurun_out/final/bench_r2.err
for c in 1 2 3 5; do python bench.py --config $c > gpurun_out/final/bench_cfg${c}_r2.json 2> gpurun_out/final/bench_cfg${c}.err; done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final/bench_ref_r2.json 2> gpurun_out/final/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/final/r2_launches_cfg4.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/final/ncu_launch.log 2>&1
bash tools/ncu_box.sh
python -m paper_1210_0084_b200.realtime --config 1 2 3 4 5 > gpurun_out/final/realtime.log 2>&1
ls gpurun_out/final
