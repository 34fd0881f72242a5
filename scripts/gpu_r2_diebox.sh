set -x
python scripts/die_map.py
for rep in 1 2; do
for v in 0 1; do
  DFLOW_GEMM_DIE_SPLIT=$v timeout 600 python scripts/gemm_power.py --seconds 4 --variants fwd,wgrad > gpurun_out/diebox_${v}_$rep.log 2>&1
  grep '"ms"' gpurun_out/diebox_${v}_$rep.log | grep -v "^{" | sed "s/^/mode$v rep$rep /"
done
done
