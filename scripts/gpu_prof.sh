set -x
# DRAM bytes + time per GEMM for raster groups 4/8/16/32 and cuBLAS (same shapes)
timeout 600 python scripts/gemm_sweep.py --groups 4,8,16,32,64 --reps 3 > gpurun_out/sweep2.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/sweep_ncu.csv python scripts/gemm_sweep.py --groups 4,8,16,32,64 --reps 3 > gpurun_out/sweep_ncu.log 2>&1; echo rc=$?
# the fused-loss forward GEMM, full set with source
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16_kernel<256, 2, 0, 1, 4>" -s 1 -c 1 -o gpurun_out/prof_loss python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo rc=$?
