set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -q -m gpu -x 2>&1 | tail -3
timeout 600 python scripts/gemm_sweep.py --groups 2,4,8 --reps 3 > gpurun_out/sweep5.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/sweep5_ncu.csv python scripts/gemm_sweep.py --groups 2,4,8 --reps 3 > gpurun_out/sweep_ncu.log 2>&1; echo rc=$?
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$?; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
