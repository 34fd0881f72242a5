set -x
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
for e in 2 3 4; do timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:\\(int\\)$e>" -s 2 -c 1 -o gpurun_out/prof_full_epi$e python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_epi$e.log 2>&1; echo epi$e rc=$?; done
