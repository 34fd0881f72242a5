set -x
timeout 1200 python -m pytest tests/test_gpu_async.py -m gpu -x -q 2>&1 | tail -3
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $T --nproc-per-node 4 --master-port 29771 bench.py --gpus 4 --async-dp 1 > gpurun_out/async2_n4.json 2> gpurun_out/async2.err; echo rc=$?
DFLOW_TIMING_BATCH=3 DFLOW_TIMELINE=gpurun_out/tla timeout 600 $T --nproc-per-node 4 --master-port 29772 bench.py --gpus 4 --async-dp 1 --steps 9 --repeats 1 > gpurun_out/tla.json 2> gpurun_out/tla.err; echo rc=$?
tail -1 gpurun_out/async2_n4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), [round(x,3) for x in d['ms_per_step_repeats']], d['clocks']['sm_mhz'], d['loss'])"
tail -3 gpurun_out/async2.err
