# evict-first epilogue traffic (args.evict): suite, interleaved A/B of C3 N=1, DRAM bytes per GEMM
set -x
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py tests/test_gpu_tf32.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -2
for rep in 1 2; do for v in 0 1; do
DFLOW_GEMM_EVICT=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ev_v${v}_r$rep.json 2> gpurun_out/ev.err; echo rc=$?
done; done
DFLOW_GEMM_EVICT=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 120 --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 3 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/ev_ncu.log 2>&1; echo ncu rc=$?
for f in gpurun_out/ev_v*.json; do echo $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), [round(x,3) for x in d['ms_per_step_repeats']], d['clocks']['sm_mhz'], d['clocks']['power_w_max'], round(d['roofline']['avg_launch_ms'],4))"); done
