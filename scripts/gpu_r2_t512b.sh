# Where the 256 x 512 pair tile loses cycles: mainloop-only (debug 2: no epilogue) and
# MMA-only (debug 3: no TMA, no epilogue) sustained runs beside the 256 x 256 tile.
mkdir -p gpurun_out/t512
timeout 900 python scripts/gemm_power.py --seconds 4 \
  --variants fwd_d2,fwd_d2_t3,fwd_d3,fwd_d3_t3,fwd_d2_t3,fwd_d2,fwd_d1_t3,fwd_d1,wgrad_d2,wgrad_d2_t3,fwd,fwd_t3 \
  > gpurun_out/t512/power_dbg.log 2>&1; tail -n 13 gpurun_out/t512/power_dbg.log | cut -c1-200
