# epilogue L2 prefetch of y / mask / W rows during the mainloop: suite, interleaved A/B C3 N=1, launch list
set -x
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py tests/test_gpu_tf32.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -2
for rep in 1 2; do for v in 0 1; do
DFLOW_GEMM_EPI_PREFETCH=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/pf_v${v}_r$rep.json 2> gpurun_out/pf.err; echo rc=$?
done; done
for v in 0 1; do
DFLOW_GEMM_EPI_PREFETCH=$v timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 60 --csv --log-file gpurun_out/pf_launches_v$v.csv python bench.py --steps 3 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/pf_ncu.log 2>&1; echo ncu rc=$?
done
for f in gpurun_out/pf_v*.json; do echo $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), [round(x,3) for x in d['ms_per_step_repeats']], d['clocks']['sm_mhz'], d['clocks']['power_w_max'], round(d['roofline']['avg_launch_ms'],4))"); done
