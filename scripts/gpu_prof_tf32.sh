set -x
timeout 900 python bench.py --config C5 --steps 1 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/bench_c5_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:\\(bool\\)1, \\(bool\\)0, \\(bool\\)1, \\(int\\)2>" -s 3 -c 1 -o gpurun_out/prof_tf32_fwd python bench.py --config C5 --steps 1 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/ncu_tf32.log 2>&1; echo rc=$?
tail -3 gpurun_out/ncu_tf32.log
