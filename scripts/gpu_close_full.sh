# one ncu --set full capture per GEMM variant of the C3 step on the closing build (EPI 3 dgrad+ReluGrad,
# EPI 4 loss-fused forward, EPI 5 wgrad+SGD; EPI 2 is profiles/r1_close/ncu_full_gemm.txt)
set -x
timeout 600 python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/e_small.log 2>&1; echo small rc=$?
for e in 3 4 5; do
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:\\(int\\)$e>" -s 1 -c 1 -o gpurun_out/e_full_epi$e python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/e_ncu_epi$e.log 2>&1; echo epi$e rc=$?
done
ls -la gpurun_out/
