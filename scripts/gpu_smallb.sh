# per-GPU GEMM efficiency at the local batches of N = 4 and N = 8 (C3 widths), one GPU
set -x
for b in 4096 8192; do
timeout 600 python bench.py --batch $b --no-cpu-baseline > gpurun_out/bench_b$b.json 2> gpurun_out/bench_b$b.err; echo rc=$?; cat gpurun_out/bench_b$b.json
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 400 --csv --log-file gpurun_out/launches_b4096.csv python bench.py --batch 4096 --steps 3 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/ncu_b4096.log 2>&1; echo ncu rc=$?
