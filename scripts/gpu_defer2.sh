set -x
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -k "DEFER" 2>&1 | tail -25
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
DFLOW_TIMELINE=gpurun_out/tld timeout 600 $T --nproc-per-node 4 --master-port 29521 bench.py --gpus 4 --repeats 1 > gpurun_out/tld.json 2> gpurun_out/tld.err; echo rc=$?
DFLOW_TIMELINE=gpurun_out/tle timeout 600 $T --nproc-per-node 4 --master-port 29522 bench.py --gpus 4 --repeats 1 --defer-apply 0 > gpurun_out/tle.json 2> gpurun_out/tle.err; echo rc=$?
timeout 600 $T --nproc-per-node 4 --master-port 29523 bench.py --gpus 4 --batch 16384 --defer-apply 0 > gpurun_out/n4_b16384_eager.json 2> gpurun_out/n4_b16384e.err; echo rc=$?; tail -1 gpurun_out/n4_b16384_eager.json | cut -c1-300
timeout 600 $T --nproc-per-node 4 --master-port 29524 bench.py --gpus 4 --batch 16384 --defer-apply 1 > gpurun_out/n4_b16384_defer2.json 2> gpurun_out/n4_b16384d.err; echo rc=$?; tail -1 gpurun_out/n4_b16384_defer2.json | cut -c1-300
