set -x
timeout 900 python -m pytest tests/test_gpu_tf32.py tests/test_gpu_kernels.py -q -m gpu -x 2>&1 | tail -2
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo rc=$?; tail -c 400 gpurun_out/bench_c5.json
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$?
