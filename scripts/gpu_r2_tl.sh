set -x
for v in r1:_r1 r2:.; do
  tag=${v%%:*}; dir=${v##*:}
  (cd $dir && DFLOW_TIMELINE=$GRAFT_REPO_ROOT/gpurun_out/tl_$tag DFLOW_TIMING_BATCH=3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 9 --warmup 5 --batch 16384 --repeats 1) > gpurun_out/tl_$tag.json 2> gpurun_out/tl_$tag.err
  ls gpurun_out/ | grep tl_
done
