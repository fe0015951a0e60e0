# round 2: compact single-CTA rerank chain; one-pass softmax (S read once from TMEM) vs two-pass
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "rerank or paged or parity_llama or slab" 2>&1 | tail -3 > gpurun_out/gpu_subset9.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0"
timeout 900 $B > gpurun_out/c4_onepass.json 2> gpurun_out/c4_onepass.err
TKV_LIB=paper_2601_08743_b200/lib/twopass/libtkv.so timeout 900 $B > gpurun_out/c4_twopass.json 2> gpurun_out/c4_twopass.err
TKV_ATTN_TRACE=gpurun_out/attn_c4_trace.bin timeout 900 python bench.py --config c4 --queries 200 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline > /dev/null 2>&1
python profiles/attn_trace.py gpurun_out/attn_c4_trace.bin > gpurun_out/attn_c4_trace.txt 2>&1
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c5_onepass.json 2> gpurun_out/c5_onepass.err
cat gpurun_out/gpu_subset9.log
