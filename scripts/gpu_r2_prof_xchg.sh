set -x
python scripts/profile_exchange_kernels.py 4 4096 > gpurun_out/r2_xk_plain.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second \
    --clock-control none --csv --kernel-name regex:"k_owner|k_colsum|k_apply|k_async|k_wait|k_sum_ranks" \
    --log-file gpurun_out/r2_xk_ncu.csv python scripts/profile_exchange_kernels.py 4 4096 > gpurun_out/r2_xk_ncu.log 2>&1
tail -3 gpurun_out/r2_xk_ncu.log
