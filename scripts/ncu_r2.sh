# r2 session-3 captures: ncu --set full of the bf16 trainer and K2 in a C4 round, plus the round's launch list
ARGS="--steps 2 --warmup 3 --no-cpu --no-c5 --no-async --no-micro --no-parity --no-quality"
ncu --set full --clock-control none --import-source on -k regex:"train_kernel|shuffle16_kernel" -s 8 -c 2 \
  -o gpurun_out/r2s3_round -f python bench.py $ARGS > gpurun_out/ncu_r2s3.log 2>&1
ncu -i gpurun_out/r2s3_round.ncu-rep --page raw --csv > gpurun_out/r2s3_round_raw.csv 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 120 --csv --log-file gpurun_out/r2s3_launches.csv \
  python bench.py $ARGS > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/r2s3_launches.csv | head -20
