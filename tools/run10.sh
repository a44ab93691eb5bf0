cd /root/repo
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu10.txt 2>&1
cd tools
timeout 400 python perf_sweep.py > ../gpurun_out/sweep10.txt 2>&1
for cfg in "128 1" "256 2"; do set -- $cfg
  FDP_FORCE_CG=$2 timeout 60 python trace_fused.py c_fc $1 none > ../gpurun_out/trace10_$1_$2.txt 2>&1
  FDP_FORCE_CG=$2 timeout 60 python trace_fused.py c_fc $1 philox >> ../gpurun_out/trace10_$1_$2.txt 2>&1
  FDP_FORCE_CG=$2 timeout 60 python trace_fused.py attn_proj $1 philox >> ../gpurun_out/trace10_$1_$2.txt 2>&1
done
cd ..
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench10.json 2> gpurun_out/bench10.err
timeout 900 python tools/layer_sweep.py > gpurun_out/layer_sweep10.jsonl 2>&1
echo done
