# A/B of the tcgen05 attention's K/V ring depths (variant libraries built by hand into lib/)
set -u
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],round(d['value'],1),round(d['attention_ms_per_step'],1),round(d['gather']['ms_per_step'],1),round(d['ms_per_step'],1))" $1 $2; }
for v in k3v2 k2v3; do TKV_LIB=$PWD/paper_2601_08743_b200/lib/libtkv_$v.so timeout 600 python -m pytest tests/test_gpu.py -x -q -k "tcgen05 or serving_path" 2>&1 | tail -1; done
for v in k2v2 k3v2 k2v3; do L=$PWD/paper_2601_08743_b200/lib/libtkv_$v.so; [ $v = k2v2 ] && L=$PWD/paper_2601_08743_b200/lib/libtkv.so
  TKV_ATTN_PREFETCH=0 TKV_LIB=$L timeout 900 python bench.py --config c5 --capacity 64 --queries 1250 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline > gpurun_out/st_c5_$v.json 2>/dev/null; show gpurun_out/st_c5_$v.json c5_$v
  TKV_ATTN_PREFETCH=0 TKV_LIB=$L timeout 900 python bench.py --no-cpu-baseline --nocache-queries 0 --steps 2 > gpurun_out/st_c2_$v.json 2>/dev/null; show gpurun_out/st_c2_$v.json c2_$v
done
