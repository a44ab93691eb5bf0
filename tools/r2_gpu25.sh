#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export FDP_NO_COOP=1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum \
  --csv --log-file gpurun_out/bytes_r2.csv python tools/bytes_moved.py > gpurun_out/bytes_r2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dpdw_group -s 2 -c 1 \
  -o gpurun_out/prof_group_r2b -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-nondp --no-train \
  > gpurun_out/prof_group_r2b.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r2b.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-train \
  > gpurun_out/launch_bench_r2b.log 2>&1
echo done
