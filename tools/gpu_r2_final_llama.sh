# Final Llama training-step numbers of round 2 (one B200): 7B B=1/2 all-reduce DP-Adam, 13B shapes 20 blocks ZeRO-1 B=1/2
mkdir -p gpurun_out
python tools/train_llama.py --model llama-7b --batch 1 --steps 4 --warmup 2 > gpurun_out/fl7_b1.json 2> gpurun_out/fl.err
python tools/train_llama.py --model llama-7b --batch 2 --steps 4 --warmup 2 > gpurun_out/fl7_b2.json 2>> gpurun_out/fl.err
python tools/train_llama.py --model llama-13b --layers 20 --zero1 --batch 1 --steps 4 --warmup 2 > gpurun_out/fl13_b1.json 2>> gpurun_out/fl.err
python tools/train_llama.py --model llama-13b --layers 20 --zero1 --batch 2 --steps 4 --warmup 2 > gpurun_out/fl13_b2.json 2>> gpurun_out/fl.err
python tools/train_llama_prof.py --model llama-7b --layers 4 > gpurun_out/fl_prof7.jsonl 2>> gpurun_out/fl.err
