# round 2: grouped paged tile layout (one 4-D TMA box per 8-row group) — tests, C4/C2/C5
set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "paged or parity or serving or executor or slab" 2>&1 | tail -5 > gpurun_out/gpu_subset19.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c4_grp.json 2> gpurun_out/c4_grp.err
timeout 900 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c2_grp.json 2> gpurun_out/c2_grp.err
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c5_grp.json 2> gpurun_out/c5_grp.err
TKV_ATTN_TRACE=gpurun_out/attn_c4_trace.bin timeout 900 python bench.py --config c4 --queries 200 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline > /dev/null 2>&1
python profiles/attn_trace.py gpurun_out/attn_c4_trace.bin > gpurun_out/attn_c4_trace.txt 2>&1
cat gpurun_out/gpu_subset19.log
