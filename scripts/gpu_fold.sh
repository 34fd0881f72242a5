set -x
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for fb in 296 148 64 32; do
DFLOW_FOLD_BLOCKS=$fb DFLOW_TIMING_BATCH=3 DFLOW_TIMELINE=gpurun_out/tf$fb timeout 600 $T --nproc-per-node 4 --master-port $((29700+fb%97)) bench.py --gpus 4 --batch 16384 --steps 9 --repeats 1 > gpurun_out/tf$fb.json 2> gpurun_out/tf.err; echo rc=$?
done
