set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 600 > gpurun_out/die2_tests.log 2>&1; tail -1 gpurun_out/die2_tests.log
DFLOW_GEMM_DIE_SPLIT=2 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -q -x --timeout 600 >> gpurun_out/die2_tests.log 2>&1; tail -1 gpurun_out/die2_tests.log
for rep in 1 2; do
for v in 0 1 2; do
  DFLOW_GEMM_DIE_SPLIT=$v timeout 600 python scripts/gemm_power.py --seconds 4 --variants fwd,dgrad,wgrad > gpurun_out/die2_power_${v}_$rep.log 2>&1
done
done
grep -H '"ms"' gpurun_out/die2_power_*.log | grep -v ':{'
