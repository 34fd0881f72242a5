set -x
ab() {  # $1 tag, $2 dir, extra args
  tag=$1; dir=$2; shift 2
  (cd $dir && timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 20 --warmup 5 "$@") > gpurun_out/ab3_$tag.json 2> gpurun_out/ab3_$tag.err
  tail -c 200 gpurun_out/ab3_$tag.json
}
for rep in 1 2; do
  ab r1_px_$rep _r1 --batch 16384
  ab r2_px_$rep . --batch 16384
  ab r1_n4_$rep _r1
  ab r2_n4_$rep .
done
