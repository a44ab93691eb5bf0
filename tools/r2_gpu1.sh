#!/bin/bash
# round 2, first GPU call: Llama-shape parity, small-T ncu captures, bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
nproc > gpurun_out/nproc.txt
timeout 1500 python -m pytest tests/test_gpu_llama_parity.py -x -q --durations=50 > gpurun_out/pytest_llama.txt 2>&1
for s in "64 128 1024 1024" "64 128 2048 2048"; do
  tag=$(echo $s | tr ' ' '_')
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:dpdw -s 2 -c 1 \
    -o gpurun_out/r2_smallT_$tag -f python tools/prof_shape.py $s fused 3 > gpurun_out/ncu_smallT_$tag.log 2>&1
done
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo done
