# DRAM bytes per GEMM launch, previous library (_abprev/) vs the pipelined epilogue, same box,
# twice each (interleaved); then the loss-fused forward's --set full capture.
O=gpurun_out/dram_ab
mkdir -p $O
for rep in 1 2; do
  for d in . _abprev; do
    tag=$( [ $d = . ] && echo cur || echo prev )
    (cd $d && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_ltcfabric.sum \
       --clock-control none --csv -c 80 --kernel-name regex:gemm_kernel --log-file /tmp/l_${tag}_$rep.csv \
       python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --c5-sub 0 > /dev/null 2>&1)
    cp /tmp/l_${tag}_$rep.csv $O/launches_${tag}_$rep.csv
  done
done
timeout 900 ncu --set full --clock-control none --import-source on \
   --kernel-name regex:"gemm_kernel<.int.256, .int.2, .bool.0, .bool.0, .bool.1, .int.4>" --launch-skip 2 --launch-count 1 \
   -o $O/gemm_loss python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --c5-sub 0 > $O/ncu_loss.log 2>&1
ncu -i $O/gemm_loss.ncu-rep --page raw --csv > $O/gemm_loss_raw.csv 2>/dev/null
ncu -i $O/gemm_loss.ncu-rep --page source --csv --print-source sass > $O/gemm_loss_src.csv 2>/dev/null
ls -la $O
