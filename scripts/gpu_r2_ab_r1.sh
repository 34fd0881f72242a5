# A/B on one 4-GPU box: round-1 HEAD (_r1/, untracked copy) vs this build, interleaved
set -x
ab() {  # $1 tag, $2 dir, $3 ngpus, extra args
  tag=$1; dir=$2; n=$3; shift 3
  if [ "$n" = 1 ]; then
    (cd $dir && timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline "$@") > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
  else
    (cd $dir && timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + RANDOM % 200)) bench.py --gpus $n --steps 20 --warmup 5 "$@") > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
  fi
  tail -c 300 gpurun_out/ab_$tag.json
}
for rep in 1 2; do
  ab r1_n4_$rep _r1 4
  ab r2_n4_$rep . 4
  ab r1_px_$rep _r1 4 --batch 16384
  ab r2_px_$rep . 4 --batch 16384
done
ab r1_n1 _r1 1
ab r2_n1 . 1 --c5-sub 0
