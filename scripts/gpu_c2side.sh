set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py tests/test_gpu_tf32.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --config C2 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/c2_side.json 2> gpurun_out/c2_side.err; echo rc=$?; tail -1 gpurun_out/c2_side.json | cut -c1-400
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/c3_side.json 2> gpurun_out/c3_side.err; echo rc=$?; tail -1 gpurun_out/c3_side.json | cut -c1-400
timeout 600 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c2_side.csv python bench.py --config C2 --steps 3 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1; echo ncu rc=$?
