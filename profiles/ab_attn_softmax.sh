# attention softmax change: parity tests, then C2 / C5 attention time
set -u
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "serving_path or edge or executor or tcgen05" 2>&1 | tail -1
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],round(d['value'],1),round(d['attention_ms_per_step'],1),round(d['gather']['ms_per_step'],1),d['gather']['gbs'],round(d['ms_per_step'],1))" $1 $2; }
timeout 900 python bench.py --no-cpu-baseline --nocache-queries 0 --steps 2 > gpurun_out/sm_c2.json 2>/dev/null; show gpurun_out/sm_c2.json c2
timeout 900 python bench.py --config c5 --capacity 64 --queries 1250 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline > gpurun_out/sm_c5.json 2>/dev/null; show gpurun_out/sm_c5.json c5
TKV_ATTN_TRACE=gpurun_out/c5trace_sm.bin timeout 900 python bench.py --config c5 --capacity 64 --queries 1250 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline > /dev/null 2>&1
