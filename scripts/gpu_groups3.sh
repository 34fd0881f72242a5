# per-kind raster group A/B on the whole C3 step (interleaved): plan default 8 everywhere vs forward group 2 / wgrad 4
set -x
run() { tag=$1; shift; env "$@" timeout 400 python bench.py --no-cpu-baseline > gpurun_out/g3_$tag.json 2> gpurun_out/g3_$tag.err
tail -1 gpurun_out/g3_$tag.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', round(d['ms_per_step'],3), [round(x,3) for x in d.get('ms_per_step_repeats',[])], d['clocks']['sm_mhz'], round(d['roofline']['kernel_ms_per_step']['gemm'],3))"; }
for i in 1 2; do
run base$i X=0
run fwd2_$i DFLOW_GEMM_GROUP_FWD=2
run fwd2w4_$i DFLOW_GEMM_GROUP_FWD=2 DFLOW_GEMM_GROUP_WGRAD=4
done
