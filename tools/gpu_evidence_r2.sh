#!/bin/bash
# Round-2 evidence for profiles/ in one gpurun call (one B200):
#   /usr/local/graft/bin/gpurun --timeout 5400 -- 'bash tools/gpu_evidence_r2.sh'
# GPU suite, bench lines (driver K/W, 200-step sustained, reference arm), ncu of the bench's
# dominant kernel + launch list, bytes moved per workflow, small-T ncu, Llama blocks / steps,
# the A/B experiments quoted in DESIGN.md.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu --no-train > gpurun_out/bench_200.json 2> gpurun_out/bench_200.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err
AB_ROUNDS=5 python tools/ab.py base FDP_PF_AHEAD=-1 FDP_PF_AHEAD=1 FDP_PAIR_DSMEM=1 > gpurun_out/ab_group.jsonl 2> gpurun_out/ab_group.err
AB_ROUNDS=3 python tools/ab_layer.py "1,2048,13824,5120;2,2048,13824,5120;1,2048,5120,5120" \
  base FDP_STREAM_SWIZZLE=0 FDP_STREAM_MC=1 > gpurun_out/ab_stream.jsonl 2> gpurun_out/ab_stream.err
python tools/llama_block.py > gpurun_out/llama_blocks.jsonl 2> gpurun_out/llama_blocks.err
python tools/train_llama.py --model llama-7b --steps 4 --warmup 2 > gpurun_out/train_llama7.json 2> gpurun_out/train_llama7.err
python tools/train_llama.py --model llama-13b --layers 20 --zero1 --steps 4 --warmup 2 > gpurun_out/train_llama13.json 2> gpurun_out/train_llama13.err
python tools/train_llama_prof.py --model llama-13b --layers 4 > gpurun_out/train_llama_prof.jsonl 2> gpurun_out/train_llama_prof.err
export FDP_NO_COOP=1   # ncu replays cannot relaunch cooperative cluster grids (co-resident either way)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-train > gpurun_out/launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dpdw_group -s 2 -c 1 -o gpurun_out/prof_group -f \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-nondp --no-train > gpurun_out/prof_group.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum \
  --csv --log-file gpurun_out/bytes.csv python tools/bytes_moved.py > gpurun_out/bytes.log 2>&1
for s in "64 128 1024 1024" "64 128 2048 2048"; do
  tag=$(echo $s | tr ' ' '_')
  ncu --set full --clock-control none --import-source on -k regex:dpdw -s 2 -c 1 -o gpurun_out/smallT_$tag -f \
    python tools/prof_shape.py $s fused 3 > gpurun_out/smallT_$tag.log 2>&1
done
echo done
