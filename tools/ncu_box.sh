#!/bin/bash
# Dev tool (GPU box): one ncu --set full capture of a cfg4 forward + inverse call, summarised
# on the box (the report itself exceeds what gpurun copies back).
R=/tmp/r2x2_cfg4
# (the warm-up call's 6 kernels are skipped: -k regex:slicq_ -s 6 -c 6)
SLICQ_PIPE=0 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:slicq_ -s 6 -c 6 \
  -o $R -f python tools/prof_once.py 4 172800000 1 > gpurun_out/ncu_x2.log 2>&1
python tools/ncu_summary.py $R.ncu-rep > gpurun_out/ncu_summary_x2.txt 2>&1
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic_x2.json
python tools/ncu_traffic.py $R.ncu-rep cfg4 gpurun_out/ncu_traffic_x2.json > /dev/null 2>&1
for k in fwd_spec "fwd_chan_kernel@0" "fwd_chan_kernel@1" "inv_chan_kernel@0" "inv_chan_kernel@1" inv_spec_persist; do
  n=$(echo $k | tr '@' '_')
  python tools/ncu_opcodes.py $R.ncu-rep ${k%@*} > gpurun_out/ncu_op_$n.txt 2>&1
  python tools/ncu_source.py $R.ncu-rep $k 40 > gpurun_out/ncu_src_$n.txt 2>&1
done
