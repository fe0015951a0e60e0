# dead second Q tile skipped (items whose tokens fit one Q tile): tests, then C2 / C5 vs the previous build
set -u
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "serving_path or tcgen05 or argmax_matches or bit_identical or edge" 2>&1 | tail -1
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],round(d['value'],1),round(d['attention_ms_per_step'],1),round(d['gather']['ms_per_step'],1),round(d['ms_per_step'],1))" $1 $2; }
for L in libtkv.so libtkv_prev.so; do
  TKV_LIB=$PWD/paper_2601_08743_b200/lib/$L timeout 900 python bench.py --no-cpu-baseline --nocache-queries 0 --steps 2 > gpurun_out/dead_c2_$L.json 2>/dev/null; show gpurun_out/dead_c2_$L.json c2_$L
  TKV_LIB=$PWD/paper_2601_08743_b200/lib/$L timeout 900 python bench.py --config c5 --capacity 64 --queries 1250 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline > gpurun_out/dead_c5_$L.json 2>/dev/null; show gpurun_out/dead_c5_$L.json c5_$L
done
