set -x
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for rep in 1 2 3; do for d in 0 1; do
i=$((i+1))
timeout 600 $T --nproc-per-node 4 --master-port $((29610+i)) bench.py --gpus 4 --batch 16384 --repeats 7 --defer-apply $d > gpurun_out/ab_d${d}_r$rep.json 2> gpurun_out/ab.err; echo rc=$?
done; done
for f in gpurun_out/ab_d*.json; do echo $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), [round(x,3) for x in d['ms_per_step_repeats']], d['clocks']['sm_mhz'])"); done
