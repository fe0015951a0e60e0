# round 2: register-window rerank chain; full GPU suite on the one-pass / paged-prefix / norm-fold build; full C4 line; C5
set -x
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gpu_suite10.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/c4_full.json 2> gpurun_out/c4_full.err
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c5.json 2> gpurun_out/c5.err
cat gpurun_out/gpu_suite10.log
