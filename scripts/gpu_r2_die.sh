set -x
python scripts/die_map.py > gpurun_out/die_map.log 2>&1; cat gpurun_out/die_map.log
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -q -x --timeout 600 > gpurun_out/die_tests.log 2>&1; tail -2 gpurun_out/die_tests.log
for v in 1 0; do
  DFLOW_GEMM_DIE_SPLIT=$v timeout 600 python scripts/gemm_power.py --seconds 4 --variants fwd,dgrad,wgrad > gpurun_out/die_power_$v.log 2>&1
done
timeout 300 python scripts/gemm_power.py --seconds 4 --variants fwd_cublas,wgrad_cublas > gpurun_out/die_power_cublas.log 2>&1
grep -h '"ms"' gpurun_out/die_power_*.log
for v in 1 0; do
  DFLOW_GEMM_DIE_SPLIT=$v ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,lts__t_sectors_srcunit_ltcfabric.sum,lts__t_sectors_srcunit_tex_op_read.sum \
     --clock-control none --csv --kernel-name regex:"gemm_kernel" --launch-skip 3 --launch-count 3 \
     --log-file gpurun_out/die_ncu_$v.csv python scripts/gemm_ncu_compare.py > /dev/null 2>&1
done
