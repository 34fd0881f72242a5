set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py tests/test_gpu_tf32.py -q -m gpu -x 2>&1 | tail -3
timeout 600 python scripts/gemm_sweep.py --groups 8 --prefetch 0,8 --debug 0 --reps 20 > gpurun_out/dbg_sweep.json 2>&1; cat gpurun_out/dbg_sweep.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/dbg_ncu.csv python scripts/gemm_sweep.py --groups 8 --prefetch 0,8 --debug 0,3 --reps 1 --no-cublas > gpurun_out/dbg_ncu.log 2>&1; echo rc=$?
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$?; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
