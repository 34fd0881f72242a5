set -x
nvidia-smi -L
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "sr16 or codec" 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -m gpu -x 2>&1 | tail -3
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29733 scripts/sr_convergence.py --steps 300 --out gpurun_out/sr_convergence.json > gpurun_out/sr_convergence.log 2>&1; echo rc=$?; tail -60 gpurun_out/sr_convergence.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29734 bench.py --gpus 4 --steps 20 --warmup 5 --exchange SR16 > gpurun_out/bench_n4_SR16_P2P.json 2> gpurun_out/bench_n4_SR16_P2P.err; echo rc=$?; cat gpurun_out/bench_n4_SR16_P2P.json
