# round-1 closing multi-GPU lines with the current build
set -x
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $T --nproc-per-node 4 --master-port 29801 bench.py --gpus 4 > gpurun_out/fm_c3_n4.json 2> gpurun_out/fm.err; echo rc=$?
timeout 600 $T --nproc-per-node 4 --master-port 29802 bench.py --gpus 4 --batch 16384 --repeats 5 > gpurun_out/fm_c3_proxy.json 2> gpurun_out/fm.err; echo rc=$?
timeout 900 $T --nproc-per-node 4 --master-port 29803 bench.py --gpus 4 --config C5 --steps 5 > gpurun_out/fm_c5_n4.json 2> gpurun_out/fm.err; echo rc=$?
timeout 900 $T --nproc-per-node 4 --master-port 29804 bench.py --gpus 4 --config C5 --batch 32768 --steps 5 > gpurun_out/fm_c5_proxy.json 2> gpurun_out/fm.err; echo rc=$?
timeout 600 $T --nproc-per-node 2 --master-port 29805 bench.py --gpus 2 > gpurun_out/fm_c3_n2.json 2> gpurun_out/fm.err; echo rc=$?
timeout 600 $T --nproc-per-node 4 --master-port 29806 bench.py --gpus 4 --exchange FP32_NCCL > gpurun_out/fm_c4_n4_fp32nccl.json 2> gpurun_out/fm.err; echo rc=$?
timeout 600 $T --nproc-per-node 4 --master-port 29807 bench.py --gpus 4 --exchange FP32 > gpurun_out/fm_c4_n4_fp32.json 2> gpurun_out/fm.err; echo rc=$?
for f in gpurun_out/fm_*.json; do echo $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), [round(x,3) for x in d['ms_per_step_repeats']], round(d['value']), d['clocks']['sm_mhz'], round(d['e2e']['value']))"); done
