#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
AB_ROUNDS=5 timeout 600 python tools/ab.py base FDP_PAIR_DSMEM=1 > gpurun_out/ab_dsmem2.jsonl 2> gpurun_out/ab_dsmem2.err
timeout 1500 python tools/train_llama.py --model llama-7b --steps 4 --warmup 2 > gpurun_out/tl7_full.json 2> gpurun_out/tl7_full.err
timeout 1500 python tools/train_llama.py --model llama-13b --layers 20 --zero1 --steps 4 --warmup 2 > gpurun_out/tl13_20.json 2> gpurun_out/tl13_20.err
timeout 900 python tools/train_llama.py --model llama-7b --layers 8 --batch 2 --steps 4 --warmup 2 > gpurun_out/tl7_8b2.json 2> gpurun_out/tl7_8b2.err
echo done
