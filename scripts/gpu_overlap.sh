N=${1:-4}
for cfg in "0 default" "8 default" "16 default" "8 8" "16 16"; do
  set -- $cfg
  R=$1; M=$2
  if [ "$M" = "default" ]; then unset NCCL_MAX_CTAS; else export NCCL_MAX_CTAS=$M; fi
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 2961$N bench.py --gpus $N --steps 30 --warmup 5 --sm-reserve $R --no-cpu-baseline > gpurun_out/ov_${R}_${M}.json 2> gpurun_out/ov_${R}_${M}.err
  python -c "import json; d=json.loads(open('gpurun_out/ov_${R}_${M}.json').read().strip().splitlines()[-1]); print('reserve $R maxctas $M', round(d['ms_per_step'],3), round(d['value']), d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done
