#!/bin/bash
# profiles for round 1 (third pass): default bench line, layer sweep, ncu of the two-phase kernels
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r1c.json 2> gpurun_out/bench_r1c.err
timeout 1200 python tools/layer_sweep.py > gpurun_out/layer_sweep_r1c.jsonl 2> gpurun_out/layer_sweep_r1c.err
export FDP_NO_COOP=1
PT_POINTS=4x2048x4096x4096 PT_PHASES=ghost timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"ghost_norm_pair|dpdw_stream" -c 2 -o gpurun_out/prof_twophase_r1c -f python tools/phase_times.py \
  > gpurun_out/prof_twophase_r1c.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r1c.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu \
  > gpurun_out/launch_bench_r1c.log 2>&1
echo done
