# quick check of the bf16 trainer: chain timing, bf16 numerics tests, config parity tests
python scripts/chain_probe.py 1 > gpurun_out/chain.txt 2>&1; grep -E "alone|full launch" gpurun_out/chain.txt
timeout 900 python -m pytest -x -q tests/test_gpu_bf16.py tests/test_gpu_configs.py ${QUICK_TESTS:-} 2>&1 | tail -3
