set -x
timeout 900 python -m pytest tests/test_gpu_step.py -q -m gpu -x 2>&1 | tail -3
timeout 600 python bench.py --config C2 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo rc=$?; cat gpurun_out/bench_c2.json; tail -3 gpurun_out/bench_c2.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$?; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
