# gather with K-only staging (half the smem per CTA): parity tests, then C2 / C5
set -u
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],round(d['value'],1),round(d['attention_ms_per_step'],1),round(d['gather']['ms_per_step'],1),round(d['gather']['gbs']),round(d['ms_per_step'],1))" $1 $2; }
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "serving_path or edge or executor or tcgen05 or gather" 2>&1 | tail -1
timeout 900 python bench.py --config c5 --capacity 64 --queries 1250 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline > gpurun_out/gs_c5.json 2>/dev/null; show gpurun_out/gs_c5.json c5
timeout 900 python bench.py --no-cpu-baseline --nocache-queries 0 --steps 2 > gpurun_out/gs_c2.json 2>/dev/null; show gpurun_out/gs_c2.json c2
