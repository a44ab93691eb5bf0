#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ddp.py tests/test_gpu_workspace_api.py -x -q > gpurun_out/pytest_ddp.txt 2>&1
timeout 600 python tools/train_llama.py --model llama-7b --layers 4 --steps 4 --warmup 2 > gpurun_out/tl7_4.json 2> gpurun_out/tl7_4.err
timeout 600 python tools/train_llama.py --model llama-13b --layers 4 --zero1 --steps 4 --warmup 2 > gpurun_out/tl13_4.json 2> gpurun_out/tl13_4.err
timeout 600 python tools/train_llama.py --model llama-7b --layers 4 --steps 4 --warmup 2 --nondp-linear torch --arms nondp > gpurun_out/tl7_4_torch.json 2> gpurun_out/tl7_4_torch.err
echo done
