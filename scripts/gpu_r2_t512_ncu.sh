# ncu source-level view of the 256 x 512 tile's forward and dgrad (where the epilogue stalls)
mkdir -p gpurun_out/t512
for v in ${VARIANTS:-fwd_t3 dgrad_t3}; do
  ncu --set full --import-source on --clock-control none --kernel-name regex:gemm_kernel --launch-skip 5 --launch-count 1 \
      -o gpurun_out/t512/ncu_$v python scripts/gemm_power.py --seconds 0.01 --variants $v > gpurun_out/t512/ncu_$v.log 2>&1
  ncu -i gpurun_out/t512/ncu_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/t512/src_$v.csv 2>/dev/null
  ncu -i gpurun_out/t512/ncu_$v.ncu-rep --page raw --csv > gpurun_out/t512/raw_$v.csv 2>/dev/null
done
ls -la gpurun_out/t512
