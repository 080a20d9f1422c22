# ncu --set full of K3 (dropout_bits_kernel) in a C4 round: pipe utilisation and stalls
ARGS="--steps 2 --warmup 3 --no-cpu --no-c5 --no-async --no-micro --no-parity --no-quality"
ncu --set full --clock-control none --import-source on -k regex:"dropout_bits_kernel" -s 3 -c 1 \
  -o gpurun_out/k3 -f python bench.py $ARGS > gpurun_out/ncu_k3.log 2>&1
ncu -i gpurun_out/k3.ncu-rep --page raw --csv > gpurun_out/k3_raw.csv 2>&1
ncu -i gpurun_out/k3.ncu-rep --page details --csv > gpurun_out/k3_details.csv 2>&1
ncu -i gpurun_out/k3.ncu-rep --page source --csv > gpurun_out/k3_src.csv 2>&1
tail -3 gpurun_out/ncu_k3.log
