# 4-GPU closing check of the final build: the multi-GPU suites; C3 at N = 1 / 2 / 4 and the 8-GPU proxy on one box;
# the reference arm under torchrun
set -x
O=gpurun_out/close4b
mkdir -p $O
timeout 2400 python -m pytest tests/test_gpu_multi.py tests/test_gpu_async.py tests/test_gpu_mp.py tests/test_gpu_concurrency.py -q -rf --timeout 900 > $O/multi_tests.txt 2>&1; tail -3 $O/multi_tests.txt
tr() {  # $1 tag, $2 n, extra
  tag=$1; n=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29800 + RANDOM % 100)) bench.py --gpus $n "$@" > $O/$tag.json 2> $O/$tag.err
  tail -c 200 $O/$tag.json
}
timeout 900 python bench.py --no-cpu-baseline --c5-sub 0 > $O/c3_n1.json 2> $O/c3_n1.err
for rep in 1 2; do
  tr c3_n2_r$rep 2
  tr c3_n4_r$rep 4
  tr proxy_r$rep 4 --batch 16384
done
timeout 900 python bench.py --no-cpu-baseline --c5-sub 0 > $O/c3_n1_b.json 2> $O/c3_n1_b.err
tr ref_n4 4 --impl reference --steps 5 --warmup 3
