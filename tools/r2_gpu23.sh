#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_all23.txt 2>&1
timeout 900 python tools/llama_block.py > gpurun_out/llama_blocks23.jsonl 2> gpurun_out/llama_blocks23.err
timeout 1500 python tools/train_llama.py --model llama-7b --steps 4 --warmup 2 > gpurun_out/tl7_full_x.json 2> gpurun_out/tl7_full_x.err
timeout 1500 python tools/train_llama.py --model llama-13b --layers 20 --zero1 --steps 4 --warmup 2 > gpurun_out/tl13_20_x.json 2> gpurun_out/tl13_20_x.err
echo done
