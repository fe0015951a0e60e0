# round 2: rerank kernel (1024 threads, word-major rows, cur in registers); K rotation from the table (A/B)
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "rerank" 2>&1 | tail -3 > gpurun_out/gpu_rerank.log
TKV_LIB=paper_2601_08743_b200/lib/krot_table/libtkv.so python scratch/cmp_paged.py '{}' '{"TKV_PAGED_K": "0"}' > gpurun_out/cmp_krot_table.json 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0"
timeout 900 $B > gpurun_out/c4_paged.json 2> gpurun_out/c4_paged.err
TKV_LIB=paper_2601_08743_b200/lib/krot_table/libtkv.so timeout 900 $B > gpurun_out/c4_krot_table.json 2> gpurun_out/c4_krot_table.err
timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c5_paged.json 2> gpurun_out/c5_paged.err
TKV_LIB=paper_2601_08743_b200/lib/krot_table/libtkv.so timeout 1200 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --nocache-queries 0 > gpurun_out/c5_krot_table.json 2> gpurun_out/c5_krot_table.err
cat gpurun_out/gpu_rerank.log gpurun_out/cmp_krot_table.json
