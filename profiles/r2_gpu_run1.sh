set -x
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
export TKV_PARITY_REPORT=gpurun_out/parity_r2.json
timeout 1500 python -m pytest tests/test_parity_llama.py -x -q -s 2>&1 | tail -30 > gpurun_out/parity_r2.log
timeout 1200 python -m pytest tests -m gpu -x -q --deselect tests/test_parity_llama.py 2>&1 | tail -15 > gpurun_out/gpu_suite_r2.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ref_c4.json 2> gpurun_out/ref_c4.err
tail -3 gpurun_out/*.log
