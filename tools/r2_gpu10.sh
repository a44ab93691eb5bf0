#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_ddp.py tests/test_gpu_workspace_api.py -q > gpurun_out/pytest_r10.txt 2>&1
timeout 900 python tools/llama_block.py --batches 1,2 > gpurun_out/llama_blocks_r2.jsonl 2> gpurun_out/llama_blocks_r2.err
timeout 600 python tools/train_llama.py --model llama-7b --layers 4 --steps 4 --warmup 2 > gpurun_out/tl7_4b.json 2> gpurun_out/tl7_4b.err
echo done
