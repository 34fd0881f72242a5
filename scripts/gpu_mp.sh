set -x
timeout 1200 python -m pytest tests/test_gpu_mp.py -q -m gpu -s 2>&1 | grep -E "^\{|passed|failed|Error|assert|^E " | tail -14
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29761 bench.py --gpus 4 --steps 10 --warmup 3 --model-parallel 1 > gpurun_out/bench_n4_mp.json 2> gpurun_out/bench_n4_mp.err; echo rc=$?; cat gpurun_out/bench_n4_mp.json; tail -5 gpurun_out/bench_n4_mp.err
