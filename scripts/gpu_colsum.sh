set -x
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_async.py tests/test_gpu_mp.py -m gpu -x -q 2>&1 | tail -4
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for rep in 1 2; do for b in 32768 16384; do
i=$((i+1))
timeout 600 $T --nproc-per-node 4 --master-port $((29540+i)) bench.py --gpus 4 --batch $b > gpurun_out/cs_n4_b${b}_r$rep.json 2> gpurun_out/cs_x.err; echo rc=$?
done; done
DFLOW_TIMELINE=gpurun_out/tlc timeout 600 $T --nproc-per-node 4 --master-port 29551 bench.py --gpus 4 --batch 16384 --repeats 1 > gpurun_out/tlc.json 2> gpurun_out/tlc.err; echo rc=$?
for f in gpurun_out/cs_n4_b*.json; do echo $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), [round(x,3) for x in d['ms_per_step_repeats']], d['clocks']['sm_mhz'])"); done
