# N = 1 step with the 256 x 512 tile off / on the weight gradient only / on everywhere
# (interleaved), then the forward's instruction counts per tile config.
mkdir -p gpurun_out/t512
for rep in 1 2 3; do
  for m in 0 2 1; do
    DFLOW_GEMM_TILE512=$m timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/t512/step_${m}_$rep.json 2> gpurun_out/t512/step_${m}_$rep.err
    python -c "import json; d=json.loads(open('gpurun_out/t512/step_${m}_$rep.json').read().strip().splitlines()[-1]); print('tile512=$m rep $rep', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], round(d['e2e']['value']))"
  done
done
for v in fwd_t3 fwd; do
  ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none \
      --kernel-name regex:gemm_kernel --launch-skip 5 --launch-count 1 --csv \
      python scripts/gemm_power.py --seconds 0.01 --variants $v 2>/dev/null | grep -E "inst_executed|duration" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
