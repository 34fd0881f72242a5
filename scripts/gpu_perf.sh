set -x
timeout 600 python scripts/gemm_sweep.py --groups 4,8,16,32 > gpurun_out/sweep.json 2>&1; cat gpurun_out/sweep.json
timeout 900 python -m pytest tests/test_gpu_step.py -q -m gpu -x 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$?; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
