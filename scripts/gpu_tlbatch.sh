# 3 consecutive steps per timeline (no per-step sync) at the 8-GPU proxy, eager vs defer
set -x
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
DFLOW_TIMING_BATCH=3 DFLOW_TIMELINE=gpurun_out/tb_e timeout 600 $T --nproc-per-node 4 --master-port 29601 bench.py --gpus 4 --batch 16384 --steps 9 --repeats 1 --defer-apply 0 > gpurun_out/tb_e.json 2> gpurun_out/tb_e.err; echo rc=$?
DFLOW_TIMING_BATCH=3 DFLOW_TIMELINE=gpurun_out/tb_d timeout 600 $T --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 --batch 16384 --steps 9 --repeats 1 --defer-apply 1 > gpurun_out/tb_d.json 2> gpurun_out/tb_d.err; echo rc=$?
tail -2 gpurun_out/tb_d.err
