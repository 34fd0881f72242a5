# closing lines: C3 N=1 (with roofline.achieved_at_timed_step), C5 N=1 (3xTF32), the reference arm at the driver's defaults
set -x
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/d_c3.json 2> gpurun_out/d_c3.err; echo rc=$?
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/d_c5.json 2> gpurun_out/d_c5.err; echo rc=$?
( time timeout 900 python bench.py --impl reference ) > gpurun_out/d_ref.json 2> gpurun_out/d_ref.err; echo ref rc=$?
tail -3 gpurun_out/d_ref.err
for f in d_c3 d_c5; do tail -1 gpurun_out/$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['ms_per_step'],3), [round(x,3) for x in d['ms_per_step_repeats']], round(d['value']), d['clocks']['sm_mhz'], round(r['achieved']), round(r['achieved_at_timed_step']), round(r['timing_pass_kernel_ms_per_step'],3))"; done
