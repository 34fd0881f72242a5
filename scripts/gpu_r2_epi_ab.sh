# The pipelined epilogue (working tree) against the previous commit's library (_abprev/):
# sustained GEMM kinds, then the N = 1 step, interleaved.
mkdir -p gpurun_out/epi_ab
for d in . _abprev . _abprev; do
  (cd $d && timeout 300 python scripts/gemm_power.py --seconds 4 --variants fwd,dgrad,wgrad 2>&1 | grep -v "^{" | sed "s|^|$d |" | cut -c1-110)
done
for rep in 1 2 3; do
  for d in . _abprev; do
    tag=$( [ $d = . ] && echo cur || echo prev )
    (cd $d && timeout 600 python bench.py --steps 30 --warmup 5) > gpurun_out/epi_ab/step_${tag}_$rep.json 2> gpurun_out/epi_ab/step_${tag}_$rep.err
    python -c "import json; d=json.loads(open('gpurun_out/epi_ab/step_${tag}_$rep.json').read().strip().splitlines()[-1]); print('$tag rep $rep', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], round(d['e2e']['value']))"
  done
done
