set -x
nvidia-smi -L
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu -x 2>&1 | tail -3
run() {  # N exchange p2p tag
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$1 --master-addr 127.0.0.1 --master-port 2961$1 bench.py --gpus $1 --steps 20 --warmup 5 --exchange $2 --p2p $3 > gpurun_out/bench_n$1_$4.json 2> gpurun_out/bench_n$1_$4.err; echo $4 rc=$?
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_n$1_$4.json').read().strip().splitlines()[-1]); print('$1 $4', d['ms_per_step'], d['value'], d['clocks'])"
}
run 4 TRUNC16 1 TRUNC16_P2P
run 4 TRUNC16 0 TRUNC16_NCCL
run 4 NONE 0 NONE
run 2 TRUNC16 1 TRUNC16_P2P
run 2 TRUNC16 0 TRUNC16_NCCL
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo rc=$?; cat gpurun_out/bench_c5.json
timeout 900 python bench.py --config C2 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo rc=$?; cat gpurun_out/bench_c2.json
