#!/bin/bash
# ncu evidence + layer sweep for profiles/ (round 1, second session)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export FDP_NO_COOP=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r1b.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu \
  > gpurun_out/launch_bench_r1b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dpdw_group -s 2 -c 1 \
  -o gpurun_out/prof_group_r1b -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-nondp \
  > gpurun_out/prof_group_r1b.log 2>&1
unset FDP_NO_COOP
timeout 1200 python tools/layer_sweep.py > gpurun_out/layer_sweep.jsonl 2> gpurun_out/layer_sweep.err
echo done
