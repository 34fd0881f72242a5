# EPI_BIAS_RELU_LOSS (last forward GEMM) diagnosis: per-launch time / tensor activity with
# DFLOW_GEMM_DEBUG = 0 (as built), 8 (targets not loaded), 2 (no epilogue work), then one
# source-level full capture of the loss GEMM as built
set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
for d in 0 8 2; do
DFLOW_GEMM_DEBUG=$d timeout 900 ncu --metrics $M --clock-control none -c 45 --csv --log-file gpurun_out/lossdbg_$d.csv python bench.py --steps 1 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/lossdbg_$d.log 2>&1; echo ncu$d rc=$?
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 20 -c 11 -o gpurun_out/prof_step_full python bench.py --steps 1 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
