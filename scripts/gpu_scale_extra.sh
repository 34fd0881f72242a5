set -x
timeout 600 python -m pytest tests/test_gpu_step.py -q -m gpu -x -k "p15 or host_fed" 2>&1 | tail -3
# §8(d) 8-GPU fallback: weak-scaling proxy = N=4 with the N=8 local batch (C3 global 16384, C5 global 32768)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29741 bench.py --gpus 4 --steps 20 --warmup 5 --batch 16384 > gpurun_out/bench_n4_c3_b16384.json 2> gpurun_out/bench_n4_c3_b16384.err; echo rc=$?; tail -c 600 gpurun_out/bench_n4_c3_b16384.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29742 bench.py --gpus 4 --config C5 --steps 10 --warmup 3 > gpurun_out/bench_n4_c5.json 2> gpurun_out/bench_n4_c5.err; echo rc=$?; tail -c 600 gpurun_out/bench_n4_c5.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29743 bench.py --gpus 4 --config C5 --steps 10 --warmup 3 --batch 32768 > gpurun_out/bench_n4_c5_b32768.json 2> gpurun_out/bench_n4_c5_b32768.err; echo rc=$?; tail -c 600 gpurun_out/bench_n4_c5_b32768.json
timeout 600 python bench.py --config C2 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 60 --csv --log-file gpurun_out/launches_c2.csv python bench.py --config C2 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1; echo ncu rc=$?
