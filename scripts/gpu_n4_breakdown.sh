set -x
for ex in TRUNC16 NONE; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 20 --warmup 5 --exchange $ex > gpurun_out/bd_n4_$ex.json 2> gpurun_out/bd_n4_$ex.err; echo rc=$?
done
