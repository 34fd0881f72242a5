# 2 GPUs: multi-GPU parity suites (multicast gather on by default), N=2 bench with / without multicast
set -x
nvidia-smi topo -m | head -5
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_async.py tests/test_gpu_mp.py tests/test_gpu_concurrency.py -q -rf --timeout 600 > gpurun_out/r2_multi2_tests.log 2>&1
tail -5 gpurun_out/r2_multi2_tests.log
for mc in 1 0; do
  DFLOW_P2P_MULTICAST=$mc timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2_n2_mc$mc.json 2> gpurun_out/r2_n2_mc$mc.err
  tail -c 600 gpurun_out/r2_n2_mc$mc.json
done
