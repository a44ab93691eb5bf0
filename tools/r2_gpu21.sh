#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_workspace_api.py tests/test_gpu_ddp.py tests/test_gpu_parity.py -q -k "adam or train_demo or workspace or report or noise or bucketed or zero1" > gpurun_out/pytest_r21.txt 2>&1
timeout 1500 python tools/train_llama.py --model llama-13b --layers 20 --zero1 --steps 4 --warmup 2 > gpurun_out/tl13_20_w.json 2> gpurun_out/tl13_20_w.err
timeout 1500 python tools/train_llama.py --model llama-13b --layers 20 --zero1 --batch 2 --steps 4 --warmup 2 > gpurun_out/tl13_20b2_w.json 2> gpurun_out/tl13_20b2_w.err
timeout 1500 python tools/train_llama.py --model llama-7b --steps 4 --warmup 2 --batch 2 > gpurun_out/tl7_full_b2.json 2> gpurun_out/tl7_full_b2.err
echo done
