# Sustained (200-step) group-kernel step with the norm all-reduce polling spinning vs backing off
# (FDP_POLL_NS): spinning warps draw power, and a long run sits at the power cap
mkdir -p gpurun_out
for rep in 1 2; do
  for ns in 0 64 256; do
    FDP_POLL_NS=$ns python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu --no-train --no-nondp --no-llama 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'poll_ns': $ns, 'rep': $rep, 'ms': d['ms_per_step'], 'frac': d['roofline']['frac'], 'clocks': d['clocks']}))"
  done
done
