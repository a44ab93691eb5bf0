# PDL evidence: full GPU suite, small-T paths, Llama B=2 steps, shared-X A/B
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1
tail -2 gpurun_out/pytest_gpu.txt
python tools/smallT_phases.py > gpurun_out/smallT_phases_pdl.jsonl 2> /dev/null
AB_PATH=two_phase AB_ROUNDS=4 python tools/ab_layer.py "2,2048,4096,4096;2,2048,4096,11008" base FDP_PDL=0 > gpurun_out/ab_pdl2.jsonl 2>/dev/null
python tools/train_llama.py --model llama-7b --batch 2 --steps 4 --warmup 2 > gpurun_out/tl7_b2_pdl.json 2> gpurun_out/tl7_b2_pdl.err
python tools/train_llama.py --model llama-13b --layers 20 --zero1 --batch 2 --steps 4 --warmup 2 > gpurun_out/tl13_b2_pdl.json 2> gpurun_out/tl13_b2_pdl.err
