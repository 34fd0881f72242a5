# C4 (BASELINE configs[3]): C3 with the 16-bit truncated exchange vs fp32 exchange, at N = 4 (the
# 8-GPU fallback) and at the 8-GPU proxy batch; interleaved repetitions on one box
set -x
O=gpurun_out/c4
mkdir -p $O
tr() {  # $1 tag, extra
  tag=$1; shift 1
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port $((29850 + RANDOM % 100)) bench.py --gpus 4 --steps 20 --warmup 5 "$@" > $O/$tag.json 2> $O/$tag.err
  tail -c 150 $O/$tag.json
}
for rep in 1 2; do
  tr t16p2p_r$rep --exchange TRUNC16
  tr t16nccl_r$rep --exchange TRUNC16 --p2p 0
  tr fp32_r$rep --exchange FP32
  tr fp32nccl_r$rep --exchange FP32_NCCL
  tr sr16_r$rep --exchange SR16
done
for rep in 1 2; do
  tr px_t16p2p_r$rep --exchange TRUNC16 --batch 16384
  tr px_fp32nccl_r$rep --exchange FP32_NCCL --batch 16384
done
