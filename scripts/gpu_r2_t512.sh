# The 256 x 512 pair tile (tile 3): exactness, then sustained A/B against the 256 x 256 pair
# tile per GEMM kind, then the N = 1 step with the wide tile on (interleaved runs).
set -x
mkdir -p gpurun_out/t512
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" 2>&1 | tail -5
timeout 900 python scripts/gemm_power.py --seconds 4 \
  --variants fwd,fwd_t3,dgrad,dgrad_t3,wgrad,wgrad_t3,fwd_t3,fwd,dgrad_t3,dgrad,wgrad_t3,wgrad \
  > gpurun_out/t512/power.log 2>&1; tail -n 14 gpurun_out/t512/power.log
for rep in 1 2; do
  DFLOW_GEMM_TILE512=0 timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/t512/bench_off_$rep.json 2> gpurun_out/t512/bench_off_$rep.err
  tail -c 300 gpurun_out/t512/bench_off_$rep.json
  DFLOW_GEMM_TILE512=1 timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/t512/bench_on_$rep.json 2> gpurun_out/t512/bench_on_$rep.err
  tail -c 300 gpurun_out/t512/bench_on_$rep.json
done
