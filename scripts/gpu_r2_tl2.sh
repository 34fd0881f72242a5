set -x
tl() {  # $1 tag, $2 dir, env...
  tag=$1; dir=$2; shift 2
  (cd $dir && env "$@" DFLOW_TIMELINE=$GRAFT_REPO_ROOT/gpurun_out/tl2_$tag DFLOW_TIMING_BATCH=3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 20 --warmup 5 --batch 16384) > gpurun_out/tl2_$tag.json 2> gpurun_out/tl2_$tag.err
  tail -c 150 gpurun_out/tl2_$tag.json
}
for rep in 1 2; do
  tl r1_$rep _r1 X=1
  tl r2mc_$rep . X=1
  tl r2uni_$rep . DFLOW_P2P_MULTICAST=0
done
