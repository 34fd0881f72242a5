# round-1 closing measurements on one GPU: bench lines (C3 with cpu_baseline, C2, C5), the
# ncu launch list of the C3 bench command and one --set full capture of the dW GEMM
set -x
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
timeout 900 python bench.py > gpurun_out/fin_c3.json 2> gpurun_out/fin_c3.err; echo rc=$?
timeout 600 python bench.py --config C2 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/fin_c2.json 2> gpurun_out/fin_c2.err; echo rc=$?
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/fin_c5.json 2> gpurun_out/fin_c5.err; echo rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/fin_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 400 --csv --log-file gpurun_out/fin_launches_c3.csv python bench.py --steps 3 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/fin_ncu1.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 12 -c 1 -o gpurun_out/fin_gemm python bench.py --steps 3 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/fin_ncu2.log 2>&1; echo ncu2 rc=$?
for f in fin_c3 fin_c2 fin_c5; do tail -1 gpurun_out/$f.json | cut -c1-250; done
