set -x
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -m gpu -x 2>&1 | tail -3
for n in 4 2; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 300)) bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/oa_n$n.json 2> gpurun_out/oa_n$n.err; echo n$n rc=$?; done
