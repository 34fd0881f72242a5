# defer_apply + one-fence grid signal: multi-GPU parity, then C3 at N = 2 / 4 and the 8-GPU proxy
set -x
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -k "DEFER or P2P" 2>&1 | tail -5
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $T --nproc-per-node 4 --master-port 29511 bench.py --gpus 4 > gpurun_out/n4_defer.json 2> gpurun_out/n4_defer.err; echo rc=$?; cat gpurun_out/n4_defer.json
timeout 600 $T --nproc-per-node 4 --master-port 29512 bench.py --gpus 4 --defer-apply 0 > gpurun_out/n4_eager.json 2> gpurun_out/n4_eager.err; echo rc=$?; cat gpurun_out/n4_eager.json
timeout 600 $T --nproc-per-node 4 --master-port 29513 bench.py --gpus 4 --batch 16384 > gpurun_out/n4_b16384_defer.json 2> gpurun_out/n4_b16384.err; echo rc=$?; cat gpurun_out/n4_b16384_defer.json
timeout 600 $T --nproc-per-node 2 --master-port 29514 bench.py --gpus 2 > gpurun_out/n2_defer.json 2> gpurun_out/n2_defer.err; echo rc=$?; cat gpurun_out/n2_defer.json
tail -3 gpurun_out/n4_defer.err
