set -x
timeout 600 python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:\(int\)4>' -s 1 -c 1 -o gpurun_out/prof_loss2 python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/ncu_loss2.log 2>&1; echo rc=$?
tail -3 gpurun_out/ncu_loss2.log
