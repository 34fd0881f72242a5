# One-B200 closing check after the pipelined epilogue: -m gpu suite, smoke, bench lines,
# ncu launch list of the bench command and one --set full capture of the dominant GEMM
set -x
O=gpurun_out/close2
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 > $O/gpu_tests.txt 2>&1; tail -3 $O/gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 900 python bench.py > $O/bench_c3_n1.json 2> $O/bench_c3_n1.err; tail -c 300 $O/bench_c3_n1.json
timeout 600 python bench.py --config C2 --steps 4000 --warmup 100 --no-cpu-baseline --c5-sub 0 > $O/bench_c2_n1.json 2> $O/bench_c2_n1.err
timeout 900 python bench.py --impl reference > $O/ref_n1.json 2> $O/ref_n1.err; tail -c 200 $O/ref_n1.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
   --clock-control none --csv -c 400 --log-file $O/launches_c3_n1.csv \
   python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --c5-sub 0 > $O/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"gemm_kernel" --launch-skip 20 --launch-count 1 \
   -o $O/gemm_full python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --c5-sub 0 > $O/ncu_full.log 2>&1
ncu -i $O/gemm_full.ncu-rep --page raw --csv > $O/gemm_full_raw.csv 2>/dev/null
ls -la $O
# the loss-fused forward (EPI 4) alone: tensor-pipe activity after the pipelined epilogue
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled \
   --kernel-name regex:"gemm_kernel<256, 2, (0|false), (0|false), (1|true), 4>" --launch-skip 2 --launch-count 1 \
   -o $O/gemm_loss python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --c5-sub 0 > $O/ncu_loss.log 2>&1
ncu -i $O/gemm_loss.ncu-rep --page raw --csv > $O/gemm_loss_raw.csv 2>/dev/null
ls -la $O
