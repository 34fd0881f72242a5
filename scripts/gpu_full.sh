set -x
nvidia-smi -L
timeout 2400 python -m pytest tests -q -m gpu -rf > gpurun_out/full_suite.log 2>&1; echo rc=$?
tail -5 gpurun_out/full_suite.log
grep -E "^FAILED|^ERROR" gpurun_out/full_suite.log | head
