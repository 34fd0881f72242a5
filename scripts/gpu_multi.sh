set -x
nvidia-smi -L
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu -s -x 2>&1 | tail -30
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo rc=$?; cat gpurun_out/bench_n2.json; tail -5 gpurun_out/bench_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 10 --warmup 3 --exchange NONE > gpurun_out/bench_n2_none.json 2>&1; echo rc=$?; cat gpurun_out/bench_n2_none.json | tail -3
