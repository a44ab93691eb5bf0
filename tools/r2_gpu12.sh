#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python tools/llama_block.py --batches 1 --models llama-7b,llama-13b > gpurun_out/lb_pf.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_chain.py -q > gpurun_out/pytest_r12.txt 2>&1
echo done
