set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 900 python scripts/gemm_power.py --seconds 4 > gpurun_out/r2_power.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_sim.py tests/test_gpu_step.py tests/test_gpu_async.py -q -x --timeout 600 > gpurun_out/r2_colsum_tests.log 2>&1
tail -3 gpurun_out/r2_colsum_tests.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --kernel-name regex:"k_colsum" \
    --log-file gpurun_out/r2_colsum_ncu.csv python scripts/profile_exchange_kernels.py 4 4096 > /dev/null 2>&1
