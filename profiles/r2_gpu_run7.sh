# round 2: paged prefix by TMA (8-row / 1-row pool boxes) + K rotation in smem — tests, C4 A/B, timeline, C5
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "paged or parity or slab or fold or serving" 2>&1 | tail -5 > gpurun_out/gpu_subset7.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0"
timeout 900 $B > gpurun_out/c4_paged.json 2> gpurun_out/c4_paged.err
TKV_PAGED_K=0 timeout 900 $B > gpurun_out/c4_slab.json 2> gpurun_out/c4_slab.err
TKV_PAGED_K=0 TKV_LIB=paper_2601_08743_b200/lib/old_attn/libtkv.so timeout 900 $B > gpurun_out/c4_oldattn.json 2> gpurun_out/c4_oldattn.err
TKV_ATTN_TRACE=gpurun_out/attn_c4_trace.bin timeout 900 python bench.py --config c4 --queries 200 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline > /dev/null 2>&1
python profiles/attn_trace.py gpurun_out/attn_c4_trace.bin > gpurun_out/attn_c4_trace.txt 2>&1
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c5_paged.json 2> gpurun_out/c5_paged.err
cat gpurun_out/gpu_subset7.log
