set -x
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:\(int\)4>' -s 1 -c 1 -o gpurun_out/prof_loss python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_loss.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:\(int\)5>' -s 2 -c 1 -o gpurun_out/prof_wgrad python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_wgrad.log 2>&1; echo rc=$?
tail -5 gpurun_out/ncu_loss.log
