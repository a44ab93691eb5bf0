# ncu --set full of our stream-K non-DP GEMM next to cuBLAS's on Llama-7B q (4096^2, B=1, T=2048)
mkdir -p gpurun_out
export FDP_NO_COOP=1
ncu --set full --clock-control none --import-source on -k regex:"dpdw|nvjet|gemm|xmma|cutlass" -c 4 -o gpurun_out/gemm_cmp -f \
  python tools/prof_gemm_cmp.py 4096 4096 1 2048 > gpurun_out/gemm_cmp.log 2>&1
ncu -i gpurun_out/gemm_cmp.ncu-rep --page raw --csv > gpurun_out/gemm_cmp_raw.csv 2>/dev/null
