N=${1:-4}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 2981$N scripts/exchange_bench.py > gpurun_out/xbench_n$N.json 2> gpurun_out/xbench_n$N.err; echo rc=$?
python -c "
import json; d=json.load(open('gpurun_out/xbench_n$N.json'))
for r in d['rows']: print(r['mode'], r['n_params'], round(r['ms'],3), 'busbw', round(r['busbw_GBps']))"
timeout 600 python -m pytest tests/test_gpu_multi.py -q -m gpu -x 2>&1 | tail -2
