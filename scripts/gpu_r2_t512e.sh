# Epilogue v3 (pairwise bf16 pack, two alternating register sets): exactness, sustained A/B,
# instruction counts of the epilogue-heavy forward.
mkdir -p gpurun_out/t512
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py tests/test_gpu_tf32.py -q -x 2>&1 | tail -3
timeout 900 python scripts/gemm_power.py --seconds 4 \
  --variants fwd_d1_t3,fwd,fwd_t3,dgrad,dgrad_t3,wgrad,wgrad_t3,fwd_t3,fwd,dgrad_t3,dgrad,wgrad_t3,wgrad \
  > gpurun_out/t512/power_v3.log 2>&1; grep -v "^{" gpurun_out/t512/power_v3.log | cut -c1-140
for v in fwd_t3 fwd_d1_t3; do
  ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none \
      --kernel-name regex:gemm_kernel --launch-skip 5 --launch-count 1 --csv \
      python scripts/gemm_power.py --seconds 0.01 --variants $v 2>/dev/null | grep -E "inst_executed|duration|per_second" | cut -c1-200
done
