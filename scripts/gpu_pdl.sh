set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -q -m gpu -x 2>&1 | tail -2
for p in 0 1; do DFLOW_PDL=$p timeout 600 python bench.py --config C2 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2_pdl$p.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_c2_pdl$p.json').read().strip().splitlines()[-1]); print('C2 pdl$p', d['ms_per_step'], d['ms_per_step_repeats'], d['value'])"; done
for p in 0 1; do DFLOW_PDL=$p timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c3_pdl$p.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_c3_pdl$p.json').read().strip().splitlines()[-1]); print('C3 pdl$p', d['ms_per_step'], d['ms_per_step_repeats'], d['value'], d['clocks']['sm_mhz'])"; done
