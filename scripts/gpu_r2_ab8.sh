set -x
ab() {  # $1 tag, $2 dir, env...
  tag=$1; dir=$2; shift 2
  (cd $dir && env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 30 --warmup 5 --repeats 5 --batch 16384) > gpurun_out/ab8_$tag.json 2> gpurun_out/ab8_$tag.err
  tail -c 100 gpurun_out/ab8_$tag.json
}
for rep in 1 2 3; do
  ab A_r1_$rep _r1 X=1
  ab C_r2default_$rep _r2lib X=1
  ab U_r2uni_$rep _r2lib DFLOW_P2P_MULTICAST=0
done
