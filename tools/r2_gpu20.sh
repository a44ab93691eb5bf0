#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_workspace_api.py tests/test_gpu_parity.py -q -k "adam or train_demo or workspace or report" > gpurun_out/pytest_r20.txt 2>&1
timeout 900 python tools/train_llama_prof.py --model llama-13b --layers 4 > gpurun_out/prof13_b1v.jsonl 2> gpurun_out/prof13_b1v.err
timeout 1500 python tools/train_llama.py --model llama-7b --steps 4 --warmup 2 > gpurun_out/tl7_full_v.json 2> gpurun_out/tl7_full_v.err
timeout 1500 python tools/train_llama.py --model llama-13b --layers 20 --zero1 --steps 4 --warmup 2 > gpurun_out/tl13_20_v.json 2> gpurun_out/tl13_20_v.err
timeout 1500 python tools/train_llama.py --model llama-13b --layers 20 --zero1 --batch 2 --steps 4 --warmup 2 > gpurun_out/tl13_20b2_v.json 2> gpurun_out/tl13_20b2_v.err
timeout 600 ncu --set full --clock-control none -k regex:"dpdw_stream|nvjet" -c 3 -o gpurun_out/gemm_cmp_down -f python tools/prof_gemm_cmp.py 13824 5120 > gpurun_out/gemm_cmp.log 2>&1
echo done
