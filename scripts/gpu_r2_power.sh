set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 900 python scripts/gemm_power.py --seconds 4 > gpurun_out/r2_power.log 2>&1
tail -3 gpurun_out/r2_power.log
