# round 2: paged K / V loaders with shuffled row addresses — parity subset, C4 A/B against the
# round-1 attention kernel (lib/old_attn: same tree, attn_tc5.cu of ac2e758), timeline
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "paged or parity or tcgen05 or serve" 2>&1 | tail -5 > gpurun_out/gpu_subset.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0"
timeout 900 $B > gpurun_out/c4_pagedk.json 2> gpurun_out/c4_pagedk.err
TKV_PAGED_K=0 timeout 900 $B > gpurun_out/c4_slab.json 2> gpurun_out/c4_slab.err
TKV_PAGED_K=0 TKV_LIB=paper_2601_08743_b200/lib/old_attn/libtkv.so timeout 900 $B > gpurun_out/c4_oldattn.json 2> gpurun_out/c4_oldattn.err
TKV_ATTN_TRACE=gpurun_out/attn_c4_trace.bin timeout 900 python bench.py --config c4 --queries 200 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline > /dev/null 2>&1
python profiles/attn_trace.py gpurun_out/attn_c4_trace.bin > gpurun_out/attn_c4_trace.txt 2>&1
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c5_pagedk.json 2> gpurun_out/c5_pagedk.err
cat gpurun_out/gpu_subset.log
