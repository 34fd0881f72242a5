set -x
ncu --set full --clock-control none --kernel-name regex:"gemm_kernel|nvjet" --launch-skip 4 --launch-count 4 -o gpurun_out/r2_cmp python scripts/gemm_ncu_compare.py > gpurun_out/r2_cmp.log 2>&1
ncu -i gpurun_out/r2_cmp.ncu-rep --page raw --csv > gpurun_out/r2_cmp_raw.csv 2>/dev/null
ls -la gpurun_out/r2_cmp*
