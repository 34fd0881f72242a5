# bulk (TMA engine) stores in the fused-exchange dW epilogue: parity, then timelines and A/B at the 8-GPU proxy
set -x
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -k "P2P" 2>&1 | tail -3
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for v in 0 1; do
DFLOW_P2P_BULK=$v DFLOW_TIMING_BATCH=3 DFLOW_TIMELINE=gpurun_out/tbb$v timeout 600 $T --nproc-per-node 4 --master-port $((29650+v)) bench.py --gpus 4 --batch 16384 --steps 9 --repeats 1 > gpurun_out/tbb$v.json 2> gpurun_out/tbb.err; echo rc=$?
done
i=0
for rep in 1 2; do for v in 0 1; do
i=$((i+1))
DFLOW_P2P_BULK=$v timeout 600 $T --nproc-per-node 4 --master-port $((29660+i)) bench.py --gpus 4 --batch 16384 --repeats 7 > gpurun_out/bulk_v${v}_r$rep.json 2> gpurun_out/bulk.err; echo rc=$?
done; done
timeout 600 $T --nproc-per-node 2 --master-port 29680 bench.py --gpus 2 > gpurun_out/bulk_n2.json 2> gpurun_out/bulk_n2.err; echo rc=$?
for f in gpurun_out/bulk_v*.json gpurun_out/bulk_n2.json; do echo $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), [round(x,3) for x in d['ms_per_step_repeats']], d['clocks']['sm_mhz'], round(d['e2e']['value']), round(d['e2e']['blocking_value']))"); done
