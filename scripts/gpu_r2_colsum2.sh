set -x
timeout 1500 python -m pytest tests/test_gpu_sim.py tests/test_gpu_step.py tests/test_gpu_kernels.py -q -x --timeout 600 > gpurun_out/colsum2_tests.log 2>&1; tail -2 gpurun_out/colsum2_tests.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --kernel-name regex:"k_colsum|k_loss_final" -c 40 \
    --log-file gpurun_out/colsum2_ncu.csv python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --c5-sub 0 > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/colsum2_ncu.csv
