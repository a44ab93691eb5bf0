#!/bin/bash
# End-of-round-2 evidence in one gpurun call: bench lines (driver-like 20 steps, default 200 steps,
# reference arm), smoke, the bench command's ncu launch list and a --set full capture of the
# dominant kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench20.json 2> gpurun_out/final_bench20.err
python bench.py > gpurun_out/final_bench_default.json 2> gpurun_out/final_bench_default.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
export FDP_NO_COOP=1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-train > gpurun_out/final_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dpdw_group -s 2 -c 1 -o gpurun_out/final_prof_group -f \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-nondp --no-train > gpurun_out/final_prof_group.log 2>&1
echo done
