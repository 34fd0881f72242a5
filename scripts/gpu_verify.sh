# re-entry check of the committed head: smoke, full GPU suite, default bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1800 python -m pytest tests -q -m gpu -x --durations=15 2>&1 | tail -30
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$?; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
