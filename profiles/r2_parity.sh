# bf16 parity at the benchmarked widths (tests/test_parity_llama.py); report -> gpurun_out/parity_r2.json
export TKV_PARITY_REPORT=gpurun_out/parity_r2.json
timeout 1800 python -m pytest tests/test_parity_llama.py -x -q -s 2>&1 | tail -40 > gpurun_out/parity_r2.log
tail -n 5 gpurun_out/parity_r2.log
