# A/B: head-major K slab (default) vs row-major (TKV_K_HEAD_MAJOR=0)
set -u
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],round(d['value'],1),round(d['attention_ms_per_step'],1),round(d['gather']['ms_per_step'],1),round(d['ms_per_step'],1))" $1 $2; }
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "serving_path or edge or executor or tcgen05" 2>&1 | tail -1
for hm in 1 0; do
  TKV_K_HEAD_MAJOR=$hm timeout 900 python bench.py --config c5 --capacity 64 --queries 1250 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline > gpurun_out/hm_c5_$hm.json 2>/dev/null; show gpurun_out/hm_c5_$hm.json c5_hm$hm
  TKV_K_HEAD_MAJOR=$hm timeout 900 python bench.py --no-cpu-baseline --nocache-queries 0 --steps 2 > gpurun_out/hm_c2_$hm.json 2>/dev/null; show gpurun_out/hm_c2_$hm.json c2_hm$hm
done
TKV_ATTN_TRACE=gpurun_out/c5trace_hm.bin timeout 900 python bench.py --config c5 --capacity 64 --queries 1250 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline > /dev/null 2>&1
