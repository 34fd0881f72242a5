set -x
timeout 900 python -m pytest tests/test_gpu_step.py -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/e2e_c3.json 2> gpurun_out/e2e_c3.err; echo rc=$?; tail -1 gpurun_out/e2e_c3.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['e2e'], d['clocks'])"
timeout 600 python bench.py --config C2 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/e2e_c2.json 2> gpurun_out/e2e_c2.err; echo rc=$?; tail -1 gpurun_out/e2e_c2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['e2e'])"
tail -3 gpurun_out/e2e_c3.err
