#!/bin/bash
# round 2 evidence run: full GPU suite, bench (20 + 200 steps), reference arm, ncu, Llama steps/blocks
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi14.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_all14.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench14.json 2> gpurun_out/bench14.err
timeout 900 python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu --no-train > gpurun_out/bench14_200.json 2> gpurun_out/bench14_200.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref14.json 2> gpurun_out/ref14.err
export FDP_NO_COOP=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-train \
  > gpurun_out/launch_bench_r2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dpdw_group -s 2 -c 1 \
  -o gpurun_out/prof_group_r2 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-nondp --no-train \
  > gpurun_out/prof_group_r2.log 2>&1
unset FDP_NO_COOP
timeout 1200 python tools/train_llama.py --model llama-7b --steps 4 --warmup 2 > gpurun_out/tl7_full.json 2> gpurun_out/tl7_full.err
timeout 1200 python tools/train_llama.py --model llama-13b --layers 20 --zero1 --steps 4 --warmup 2 > gpurun_out/tl13_20.json 2> gpurun_out/tl13_20.err
timeout 1200 python tools/llama_block.py > gpurun_out/llama_blocks14.jsonl 2> gpurun_out/llama_blocks14.err
echo done
