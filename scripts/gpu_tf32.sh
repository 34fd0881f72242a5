set -x
timeout 600 python -m pytest tests/test_gpu_tf32.py -q -m gpu -x -s 2>&1 | tail -30
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -q -m gpu -x 2>&1 | tail -3
