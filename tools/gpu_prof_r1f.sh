#!/bin/bash
# ncu evidence for profiles/ (round 1, final session): launch list of the bench command
# and one --set full capture of the dominant kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export FDP_NO_COOP=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r1f.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-train \
  > gpurun_out/launch_bench_r1f.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dpdw_group -s 2 -c 1 \
  -o gpurun_out/prof_group_r1f -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-nondp --no-train \
  > gpurun_out/prof_group_r1f.log 2>&1
echo done
