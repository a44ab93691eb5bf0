#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python tools/train_llama_prof.py --model llama-13b --layers 4 > gpurun_out/prof13_b1.jsonl 2> gpurun_out/prof13_b1.err
timeout 900 python tools/train_llama_prof.py --model llama-13b --layers 4 --batch 2 > gpurun_out/prof13_b2.jsonl 2> gpurun_out/prof13_b2.err
echo done
