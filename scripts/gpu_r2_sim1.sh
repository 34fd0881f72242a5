set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 1500 python -m pytest tests/test_gpu_sim.py -q -rf --timeout 600 2>&1 | tail -60 > gpurun_out/r2_sim1.log
timeout 900 python -m pytest tests -m gpu -q -x --ignore=tests/test_gpu_sim.py 2>&1 | tail -30 > gpurun_out/r2_gpu_rest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
