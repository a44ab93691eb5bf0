#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_llama_parity.py tests/test_gpu_random.py tests/test_gpu_ddp.py -q -x > gpurun_out/pytest_r15.txt 2>&1
AB_ROUNDS=5 timeout 600 python tools/ab.py base > gpurun_out/ab_dsmem.jsonl 2> gpurun_out/ab_dsmem.err
timeout 1200 python tools/train_llama.py --model llama-7b --steps 4 --warmup 2 > gpurun_out/tl7_full.json 2> gpurun_out/tl7_full.err
timeout 1200 python tools/train_llama.py --model llama-13b --layers 20 --zero1 --steps 4 --warmup 2 > gpurun_out/tl13_20.json 2> gpurun_out/tl13_20.err
echo done
