set -x
R1LIKE="DFLOW_AB_LAZY_LOSS=1 DFLOW_AB_OLD_COLSUM=1 DFLOW_AB_UNBOUNDED_WAIT=1 DFLOW_AB_SHARED_SCHED=1 DFLOW_P2P_MULTICAST=0"
ab() {  # $1 tag, $2 dir, env...
  tag=$1; dir=$2; shift 2
  (cd $dir && env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 30 --warmup 5 --repeats 5 --batch 16384) > gpurun_out/ab7_$tag.json 2> gpurun_out/ab7_$tag.err
  tail -c 100 gpurun_out/ab7_$tag.json
}
for rep in 1 2 3; do
  ab B_r1like_$rep _r2lib $R1LIKE
  ab F_alwaysAR_$rep _r2lib $R1LIKE DFLOW_AB_LAZY_LOSS=0
  ab G_boundedwait_$rep _r2lib $R1LIKE DFLOW_AB_UNBOUNDED_WAIT=0
  ab H_ownsched_$rep _r2lib $R1LIKE DFLOW_AB_SHARED_SCHED=0
done
