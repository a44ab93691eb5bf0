#!/bin/bash
# One gpurun call: GPU parity suite, smoke, default bench, reference arm.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
timeout 300 python __graft_entry__.py > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 4 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/smoke.txt | tail -2; cat gpurun_out/bench.json gpurun_out/bench_ref.json
