# full -m gpu suite, smoke, one bench line (C3 N=1 + the C5 sub-measurement)
set -x
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/r2_gpu_all.log 2>&1
tail -5 gpurun_out/r2_gpu_all.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2_bench_c3.json 2> gpurun_out/r2_bench_c3.err
tail -c 3000 gpurun_out/r2_bench_c3.json
