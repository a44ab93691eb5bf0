cd tools
timeout 120 python gpu_diag.py fused_small fused_c1 fused_c1_noise fused_ragged fused_gpt2_fc fused_gpt2_attnproj > ../gpurun_out/diag8.txt 2>&1
cd ..
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu8.txt 2>&1
cd tools
timeout 400 python perf_sweep.py > ../gpurun_out/sweep8.txt 2>&1
for cfg in "128 1" "256 2"; do set -- $cfg
  FDP_FORCE_CG=$2 timeout 60 python trace_fused.py c_fc $1 none > ../gpurun_out/trace8_$1_$2.txt 2>&1
  FDP_FORCE_CG=$2 timeout 60 python trace_fused.py c_fc $1 philox >> ../gpurun_out/trace8_$1_$2.txt 2>&1
  FDP_FORCE_CG=$2 timeout 60 python trace_fused.py attn_proj $1 philox >> ../gpurun_out/trace8_$1_$2.txt 2>&1
done
echo done
