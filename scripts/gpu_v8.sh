# 256-bit epilogue accesses (DFLOW_GEMM_V8): GEMM/step suites, interleaved C3 N=1 A/B, launch list
set -x
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py tests/test_gpu_tf32.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/v8_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/v8_tests.log
for rep in 1 2; do for v in 1 0; do
DFLOW_GEMM_V8=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/v8_v${v}_r$rep.json 2> gpurun_out/v8.err; echo rc=$?
done; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
DFLOW_GEMM_V8=1 timeout 900 ncu --metrics $M --clock-control none -c 45 --csv --log-file gpurun_out/v8_launches.csv python bench.py --steps 1 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/v8_ncu.log 2>&1; echo ncu rc=$?
for f in gpurun_out/v8_v*.json; do echo $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), [round(x,3) for x in d['ms_per_step_repeats']], d['clocks']['sm_mhz'], d['clocks']['power_w_max'], round(d['roofline']['avg_launch_ms'],4))"); done
