set -x
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for rep in 1 2; do
for v in "A hi 0" "B hi 148" "C lo 148" "D lo 0"; do set -- $v
i=$((i+1))
DFLOW_COMM_PRIO=$2 DFLOW_FOLD_BLOCKS=$3 timeout 600 $T --nproc-per-node 4 --master-port $((29560+i)) bench.py --gpus 4 --batch 16384 --repeats 3 > gpurun_out/pr_$1_r$rep.json 2> gpurun_out/pr_x.err; echo rc=$?
done; done
for f in gpurun_out/pr_*.json; do echo $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), [round(x,3) for x in d['ms_per_step_repeats']], d['clocks']['sm_mhz'])"); done
