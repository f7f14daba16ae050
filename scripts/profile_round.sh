#!/usr/bin/env bash
# Run on the GPU box (under gpurun).  Produces, in gpurun_out/:
#   launches.csv      every launch of a short bench run with its device time (cold, serialised)
#   prof_fwd.ncu-rep  ncu --set full of the forward pair kernel (first timed step)
#   prof_bwd.ncu-rep  ncu --set full of the backward pair kernel (first timed step)
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_bench.json 2>&1
echo "launches rc=$?"
# the bench's sanity step uses warmup launches; pair kernel launches: 2 per step -> skip 3 warmup steps (6)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cce_pair_kernel -s 6 -c 1 \
  -o gpurun_out/prof_fwd python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "fwd rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cce_pair_kernel -s 7 -c 1 \
  -o gpurun_out/prof_bwd python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "bwd rc=$?"
# design B (CCE_FLAG_DESIGN_B): launch list and one full capture of each mode
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_designb.csv python bench.py --steps 2 --warmup 3 --flags 2048 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cce_designb_kernel -s 6 -c 2 \
  -o gpurun_out/prof_designb python bench.py --steps 1 --warmup 3 --flags 2048 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "designb rc=$?"
