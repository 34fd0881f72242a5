# round-1 closing check of HEAD on one GPU: the whole -m gpu suite, smoke(), the default bench
# line (with cpu_baseline), the reference arm, the ncu launch list and one --set full GEMM capture
set -x
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/c_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/c_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c_smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/c_smoke.log
timeout 900 python bench.py > gpurun_out/c_c3.json 2> gpurun_out/c_c3.err; echo rc=$?
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/c_ref.json 2> gpurun_out/c_ref.err; echo ref rc=$?
timeout 600 python bench.py --config C2 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/c_c2.json 2> gpurun_out/c_c2.err; echo rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 400 --csv --log-file gpurun_out/c_launches_c3.csv python bench.py --steps 3 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/c_ncu1.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 12 -c 1 -o gpurun_out/c_gemm python bench.py --steps 3 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/c_ncu2.log 2>&1; echo ncu2 rc=$?
for f in c_c3 c_ref c_c2; do tail -1 gpurun_out/$f.json | cut -c1-300; done
