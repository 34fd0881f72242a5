set -x
nvidia-smi -L
N=${1:-4}
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu -x 2>&1 | tail -3
for ex in TRUNC16 FP32 FP32_NCCL NONE; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --steps 20 --warmup 5 --exchange $ex > gpurun_out/bench_n${N}_$ex.json 2> gpurun_out/bench_n${N}_$ex.err; echo $ex rc=$?
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_n${N}_$ex.json').read().strip().splitlines()[-1]); print('$ex', d['ms_per_step'], d['value'], d['clocks'])"
done
