#!/bin/bash
# One gpurun call: tests, perf sweep, bench, launch list, one full ncu capture.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
if [ -z "$SKIP_TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1
fi
timeout 600 python tools/perf_sweep.py > gpurun_out/sweep.txt 2>&1
timeout 600 python bench.py --steps ${STEPS:-100} --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ -z "$SKIP_NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"dpdw|k_|gemm|nvjet|cutlass" -c 200 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-nondp > /dev/null 2> gpurun_out/ncu_launch.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dpdw_tc -s 2 -c 1 \
    -o gpurun_out/prof_fused_cfc -f python tools/prof_one.py c_fc 3 > gpurun_out/ncu_full.log 2>&1
fi
echo done
