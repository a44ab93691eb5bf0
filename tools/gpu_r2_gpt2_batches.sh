# GPT-2 small training step, DP vs non-DP, at the paper's batch sizes (B = 1/2/4/8, seq 1024)
mkdir -p gpurun_out
for B in 1 2 4 8; do
  python tools/train_gpt2.py --batch $B --steps 100 --warmup 10 >> gpurun_out/gpt2_batches.jsonl 2>/dev/null
  python tools/train_gpt2.py --batch $B --steps 100 --warmup 10 --full >> gpurun_out/gpt2_batches.jsonl 2>/dev/null
done
