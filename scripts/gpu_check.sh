set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 120 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "test_gemm_layouts_exact_integers and 128-128-64" -x 2>&1 | tail -30
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu 2>&1 | tail -60 > gpurun_out/kernels.log; tail -60 gpurun_out/kernels.log
timeout 600 python -m pytest tests/test_gpu_step.py -q -m gpu -s 2>&1 | tail -80 > gpurun_out/step.log; tail -80 gpurun_out/step.log
