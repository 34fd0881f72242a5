set -x
nvidia-smi -L
timeout 1200 python -m pytest tests/test_gpu_async.py -q -m gpu -s 2>&1 | grep -E "^\{|passed|failed|Error|assert" | tail -12
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -4
