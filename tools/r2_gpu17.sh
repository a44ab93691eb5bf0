#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for bn in 256 128; do timeout 120 python tools/trace_fused.py 1024x1024 $bn none 64 128 > gpurun_out/trace_t128_$bn.json 2>&1; done
timeout 120 python tools/trace_fused.py 1024x1024 256 none 16 512 > gpurun_out/trace_t512.json 2>&1
timeout 1500 python tools/train_llama.py --model llama-13b --layers 20 --zero1 --batch 2 --steps 4 --warmup 2 > gpurun_out/tl13_20b2.json 2> gpurun_out/tl13_20b2.err
echo done
