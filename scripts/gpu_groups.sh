set -x
timeout 600 python scripts/gemm_sweep.py --groups 2,4,8,16,32 --prefetch 0 --reps 10 --no-cublas > gpurun_out/grp_sweep.json 2>&1; cat gpurun_out/grp_sweep.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/grp_ncu.csv python scripts/gemm_sweep.py --groups 2,4,8,16,32 --prefetch 0 --reps 1 --no-cublas > gpurun_out/grp_ncu.log 2>&1; echo rc=$?
