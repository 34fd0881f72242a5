set -x
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo rc=$?; cat gpurun_out/bench_c3.json; tail -3 gpurun_out/bench_c3.err
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo rc=$?; cat gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5.err
timeout 900 python bench.py --config C2 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo rc=$?; cat gpurun_out/bench_c2.json; tail -3 gpurun_out/bench_c2.err
