set -x
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -k "DEFER" 2>&1 | tail -3
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for rep in 1 2; do for d in 1 0; do for b in 32768 16384; do
i=$((i+1))
timeout 600 $T --nproc-per-node 4 --master-port $((29530+i)) bench.py --gpus 4 --batch $b --defer-apply $d --repeats 3 > gpurun_out/n4_b${b}_d${d}_r$rep.json 2> gpurun_out/n4_x.err; echo rc=$?
done; done; done
for f in gpurun_out/n4_b*_d*_r*.json; do echo $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), [round(x,3) for x in d['ms_per_step_repeats']], d['clocks']['sm_mhz'])"); done
