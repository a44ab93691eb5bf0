#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 python tools/trace_fused.py 1024x1024 256 none 64 128 > gpurun_out/trace2_t128.json 2>&1
timeout 120 python tools/trace_fused.py 1024x1024 256 none 16 512 > gpurun_out/trace2_t512.json 2>&1
AB_ROUNDS=5 timeout 600 python tools/ab.py base > gpurun_out/ab_cf.jsonl 2> gpurun_out/ab_cf.err
timeout 600 python tools/smallT.py > gpurun_out/smallT2.jsonl 2> gpurun_out/smallT2.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_gpu_llama_parity.py -q -x > gpurun_out/pytest_r18.txt 2>&1
echo done
