# ncu --set full of the bf16 trainer running the C4 world's longest client alone
CHAIN_SINGLE=1 ncu --set full --clock-control none --import-source on -k regex:train_kernel -s 2 -c 1 \
  -o gpurun_out/chain_single -f python scripts/chain_probe.py > gpurun_out/ncu_chain.log 2>&1
ncu -i gpurun_out/chain_single.ncu-rep --page raw --csv > gpurun_out/chain_single_raw.csv 2>&1
ncu -i gpurun_out/chain_single.ncu-rep --page source --csv --print-source sass > gpurun_out/chain_single_src.csv 2>&1
ncu -i gpurun_out/chain_single.ncu-rep --page details --csv > gpurun_out/chain_single_details.csv 2>&1
tail -3 gpurun_out/ncu_chain.log
