#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python tools/llama_block.py --batches 1 --models llama-7b > gpurun_out/lb_ef1.jsonl 2>&1
FDP_FIN_EPI=0 timeout 600 python tools/llama_block.py --batches 1 --models llama-7b > gpurun_out/lb_ef0.jsonl 2>&1
echo done
