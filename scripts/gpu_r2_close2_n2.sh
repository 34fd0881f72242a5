# 2 GPUs, final build: the multi-GPU parity suites and one C3 N = 2 bench line
O=gpurun_out/close2_n2
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_async.py tests/test_gpu_mp.py tests/test_gpu_concurrency.py -q -rf --timeout 600 > $O/multi_tests.log 2>&1
tail -3 $O/multi_tests.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 > $O/c3_n2.json 2> $O/c3_n2.err
tail -n1 $O/c3_n2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['clocks'])"
