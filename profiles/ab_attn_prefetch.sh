set -u
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "serving_path or edge or executor or tcgen05" 2>&1 | tail -1
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],round(d['value'],1),round(d['attention_ms_per_step'],1),round(d['gather']['ms_per_step'],1),round(d['ms_per_step'],1))" $1 $2; }
for pf in 0 4 2; do TKV_ATTN_PREFETCH=$pf timeout 900 python bench.py --no-cpu-baseline --nocache-queries 0 --steps 2 > gpurun_out/ab_c2_$pf.json 2>/dev/null; show gpurun_out/ab_c2_$pf.json c2_pf$pf; done
for pf in 0 4 2; do TKV_ATTN_PREFETCH=$pf timeout 900 python bench.py --config c5 --capacity 64 --queries 1250 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline > gpurun_out/ab_c5_$pf.json 2>/dev/null; show gpurun_out/ab_c5_$pf.json c5_pf$pf; done
TKV_ATTN_TRACE=gpurun_out/c5trace_pf.bin timeout 900 python bench.py --config c5 --capacity 64 --queries 1250 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline > /dev/null 2>&1
