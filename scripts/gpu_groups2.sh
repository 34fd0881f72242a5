# tile-raster group sweep on the dynamic-scheduler build: per GEMM shape standalone, then the whole C3 step
set -x
timeout 500 python scripts/gemm_sweep.py --groups 2,4,8,16 --prefetch 0 --reps 10 --no-cublas > gpurun_out/g2_sweep.json 2>&1; echo sweep rc=$?
for g in 4 8 16; do
DFLOW_GEMM_GROUP=$g timeout 400 python bench.py --no-cpu-baseline > gpurun_out/g2_c3_g$g.json 2> gpurun_out/g2_c3_g$g.err; echo g$g rc=$?
tail -1 gpurun_out/g2_c3_g$g.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('g$g', round(d['ms_per_step'],3), [round(x,3) for x in d.get('ms_per_step_repeats',[])], d['clocks']['sm_mhz'])"
done
cat gpurun_out/g2_sweep.json | tail -40
