set -x
DFLOW_TIMELINE=gpurun_out/tl4 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 300)) bench.py --gpus 4 --steps 20 --warmup 5 --repeats 1 > gpurun_out/tl4.json 2> gpurun_out/tl4.err; echo rc=$?
DFLOW_TIMELINE=gpurun_out/tl1 timeout 900 python bench.py --steps 20 --warmup 5 --repeats 1 --no-cpu-baseline > gpurun_out/tl1.json 2> gpurun_out/tl1.err; echo rc=$?
