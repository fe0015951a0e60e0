# round 2: per-sequence first segment (no binary search per item in the paged issuers) — tests, C2/C4, C2 timeline
set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "paged or parity or serving or executor" 2>&1 | tail -3 > gpurun_out/gpu_subset17.log
timeout 900 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c2_seg0.json 2> gpurun_out/c2_seg0.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c4_seg0.json 2> gpurun_out/c4_seg0.err
TKV_ATTN_TRACE=gpurun_out/attn_c2_trace.bin timeout 900 python bench.py --config c2 --queries 200 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline > /dev/null 2>&1
python profiles/attn_trace.py gpurun_out/attn_c2_trace.bin > gpurun_out/attn_c2_trace.txt 2>&1
cat gpurun_out/gpu_subset17.log
