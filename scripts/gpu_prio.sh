N=${1:-4}
for ex in TRUNC16 NONE; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 2971$N bench.py --gpus $N --steps 30 --warmup 5 --exchange $ex --no-cpu-baseline > gpurun_out/prio_$ex.json 2> gpurun_out/prio_$ex.err
  python -c "import json; d=json.loads(open('gpurun_out/prio_$ex.json').read().strip().splitlines()[-1]); print('$ex', round(d['ms_per_step'],3), round(d['value']), d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done
