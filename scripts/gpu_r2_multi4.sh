# 4 GPUs: N=4 parity suites; C3 N=4 and the 8-GPU proxy (N=4 at the N=8 per-GPU batch),
# multicast gather on / off, interleaved
set -x
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_async.py tests/test_gpu_mp.py -q -rf --timeout 600 -k "four or 4" > gpurun_out/r2_multi4_tests.log 2>&1
tail -4 gpurun_out/r2_multi4_tests.log
run() {  # $1 tag, $2 multicast, extra args
  tag=$1; mc=$2; shift 2
  DFLOW_P2P_MULTICAST=$mc timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port $((29600 + RANDOM % 200)) bench.py --gpus 4 --steps 20 --warmup 5 "$@" > gpurun_out/r2_n4_$tag.json 2> gpurun_out/r2_n4_$tag.err
  tail -c 400 gpurun_out/r2_n4_$tag.json
}
for rep in 1 2; do
  run c3_mc1_r$rep 1
  run c3_mc0_r$rep 0
  run proxy_mc1_r$rep 1 --batch 16384
  run proxy_mc0_r$rep 0 --batch 16384
done
