N=${1:-2}
nvidia-smi -L | head -2
timeout 400 python -m pytest tests/test_gpu_multi.py -q -m gpu -x -k "P2P" -s 2>&1 | tail -6
for p in 1 0; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 2991$N bench.py --gpus $N --steps 30 --warmup 5 --p2p $p --no-cpu-baseline > gpurun_out/p2p_${N}_$p.json 2> gpurun_out/p2p_${N}_$p.err
  python -c "import json; d=json.loads(open('gpurun_out/p2p_${N}_$p.json').read().strip().splitlines()[-1]); print('p2p $p', d['config']['exchange'], round(d['ms_per_step'],3), round(d['value']), d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])" || tail -20 gpurun_out/p2p_${N}_$p.err
done
