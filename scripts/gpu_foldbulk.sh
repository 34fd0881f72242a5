set -x
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -k "P2P" 2>&1 | tail -3
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
DFLOW_TIMING_BATCH=3 DFLOW_TIMELINE=gpurun_out/tfb timeout 600 $T --nproc-per-node 4 --master-port 29731 bench.py --gpus 4 --batch 16384 --steps 9 --repeats 1 > gpurun_out/tfb.json 2> gpurun_out/tfb.err; echo rc=$?
for rep in 1 2; do
timeout 600 $T --nproc-per-node 4 --master-port $((29740+rep)) bench.py --gpus 4 --batch 16384 --repeats 7 > gpurun_out/fb_r$rep.json 2> gpurun_out/fb.err; echo rc=$?
done
timeout 600 $T --nproc-per-node 4 --master-port 29745 bench.py --gpus 4 --repeats 5 > gpurun_out/fb_c3.json 2> gpurun_out/fb.err; echo rc=$?
for f in gpurun_out/fb_*.json; do echo $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), [round(x,3) for x in d['ms_per_step_repeats']], d['clocks']['sm_mhz'], round(d['e2e']['value']))"); done
