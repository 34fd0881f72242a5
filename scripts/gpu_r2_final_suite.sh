# Final code: the whole -m gpu suite and smoke on one B200
O=gpurun_out/final
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 > $O/gpu_tests.txt 2>&1; tail -3 $O/gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
