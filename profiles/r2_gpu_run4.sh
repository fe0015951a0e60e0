# round 2: paged K (rotated in smem) + coalesced paged V — GPU suite, C4/C5 A/B vs the K-slab gather, C4 timeline
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gpu_suite.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0"
timeout 900 $B > gpurun_out/c4_pagedk.json 2> gpurun_out/c4_pagedk.err
TKV_PAGED_K=0 timeout 900 $B > gpurun_out/c4_slab.json 2> gpurun_out/c4_slab.err
TKV_LIB=paper_2601_08743_b200/lib/k2/libtkv.so timeout 900 $B > gpurun_out/c4_pagedk_k2.json 2> gpurun_out/c4_pagedk_k2.err
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c5_pagedk.json 2> gpurun_out/c5_pagedk.err
TKV_ATTN_TRACE=gpurun_out/attn_c4_trace.bin timeout 900 python bench.py --config c4 --queries 200 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline > /dev/null 2>&1
python profiles/attn_trace.py gpurun_out/attn_c4_trace.bin > gpurun_out/attn_c4_trace.txt 2>&1
cat gpurun_out/gpu_suite.log
