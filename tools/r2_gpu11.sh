#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_ddp.py tests/test_gpu_workspace_api.py -q > gpurun_out/pytest_r11.txt 2>&1
timeout 600 python tools/llama_block.py --batches 1 --models llama-7b > gpurun_out/lb_epi1.jsonl 2>&1
FDP_FIN_EPI=0 timeout 600 python tools/llama_block.py --batches 1 --models llama-7b > gpurun_out/lb_epi0.jsonl 2>&1
echo done
