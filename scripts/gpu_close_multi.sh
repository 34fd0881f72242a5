# round-1 closing check of HEAD on 4 GPUs: the multi-GPU -m gpu suites (N = 2 and 4), smoke
# with all GPUs visible, and the C3 bench lines at N = 2 / 4 / the 8-GPU proxy
set -x
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_async.py tests/test_gpu_mp.py -m gpu -q -x > gpurun_out/cm_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/cm_tests.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $T --nproc-per-node 2 --master-port 29811 bench.py --gpus 2 > gpurun_out/cm_c3_n2.json 2> gpurun_out/cm.err; echo rc=$?
timeout 600 $T --nproc-per-node 4 --master-port 29812 bench.py --gpus 4 > gpurun_out/cm_c3_n4.json 2> gpurun_out/cm.err; echo rc=$?
timeout 600 $T --nproc-per-node 4 --master-port 29813 bench.py --gpus 4 --batch 16384 --repeats 5 > gpurun_out/cm_c3_proxy.json 2> gpurun_out/cm.err; echo rc=$?
timeout 600 $T --nproc-per-node 2 --master-port 29814 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/cm_ref_n2.json 2> gpurun_out/cm_ref.err; echo ref rc=$?
for f in gpurun_out/cm_c3_*.json; do echo $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), [round(x,3) for x in d['ms_per_step_repeats']], round(d['value']), d['clocks']['sm_mhz'], round(d['e2e']['value']))"); done
