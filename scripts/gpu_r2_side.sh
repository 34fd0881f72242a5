set -x
for rep in 1 2 3; do
  for v in 0 1; do
    DFLOW_BWD_SIDE=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --c5-sub 0 > gpurun_out/side_${v}_$rep.json 2> gpurun_out/side_${v}_$rep.err
    tail -c 100 gpurun_out/side_${v}_$rep.json
  done
done
