# What the 256 x 512 tile's epilogue drain is made of: MMA + epilogue without TMA traffic
# (debug 1, unthrottled) with the output stores (16) and / or the bias broadcast (32) removed
mkdir -p gpurun_out/t512
timeout 900 python scripts/gemm_power.py --seconds 3 \
  --variants fwd_d3_t3,fwd_d1_t3,fwd_d17_t3,fwd_d33_t3,fwd_d49_t3,dgrad_d1_t3,dgrad_d17_t3,fwd_d1,fwd_d17 \
  > gpurun_out/t512/drain.log 2>&1; grep -v "^{" gpurun_out/t512/drain.log | cut -c1-150
