# Pipelined epilogue (TMEM load + streamed operand one chunk ahead, bias in lane registers):
# exactness, then sustained A/B of the 256 x 512 and 256 x 256 tiles.
mkdir -p gpurun_out/t512
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -q -x 2>&1 | tail -3
timeout 900 python scripts/gemm_power.py --seconds 4 \
  --variants fwd_d1,fwd_d1_t3,fwd,fwd_t3,dgrad,dgrad_t3,wgrad,wgrad_t3,fwd_t3,fwd,dgrad_t3,dgrad,wgrad_t3,wgrad \
  > gpurun_out/t512/power_pipe.log 2>&1; grep -v "^{" gpurun_out/t512/power_pipe.log | cut -c1-140
