set -x
timeout 3000 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/r2_full2.log 2>&1
tail -6 gpurun_out/r2_full2.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke2.log 2>&1; tail -2 gpurun_out/r2_smoke2.log
