# ncu --set full of one factored fwd and one bwd launch of the C5 share round, per library variant
cp paper_2503_15448_b200/_fedsim_b200.so /tmp/cur.so
for v in ${VARIANTS}; do
  cp $v paper_2503_15448_b200/_fedsim_b200.so
  n=$(basename $v .so)
  ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|bwd_kernel" -s 60 -c 1 -o gpurun_out/wide_$n -f \
    python scripts/c5_only.py 1 > /dev/null 2>&1
  ncu -i gpurun_out/wide_$n.ncu-rep --page raw --csv > gpurun_out/wide_${n}_raw.csv 2>&1
done
cp /tmp/cur.so paper_2503_15448_b200/_fedsim_b200.so
for v in ${VARIANTS}; do
  n=$(basename $v .so)
  ncu -i gpurun_out/wide_$n.ncu-rep --page source --csv --print-source sass > gpurun_out/wide_${n}_src.csv 2>&1
done
