set -x
for p in 256 128 64 0; do
  DFLOW_GEMM_L2PROMO=$p timeout 600 python scripts/gemm_power.py --seconds 4 --variants fwd,dgrad,wgrad > gpurun_out/r2_promo_$p.log 2>&1
done
timeout 300 python scripts/gemm_power.py --seconds 4 --variants fwd_cublas,wgrad_cublas > gpurun_out/r2_promo_cublas.log 2>&1
grep -h '"ms"' gpurun_out/r2_promo_*.log
