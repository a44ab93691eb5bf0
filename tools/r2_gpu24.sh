#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
start=$(date +%s)
python bench.py --steps 20 --warmup 5 > gpurun_out/bench24.json 2> gpurun_out/bench24.err
end=$(date +%s)
echo "bench wall $((end-start)) s" > gpurun_out/bench24.wall
echo done
