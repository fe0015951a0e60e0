# RMSNorm folded into the GEMM epilogues (default) vs the norm kernel (TKV_NORM_FOLD=0)
set -u
timeout 1200 python -m pytest tests/test_gpu.py -q -m gpu -k "bf16 or serving_path or executor or tcgen05 or bit_identical or edge" 2>&1 | tail -3
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],round(d['value'],1),round(d['e2e']['value'],1),round(d['ms_per_step'],1),d['roofline']['frac'],d['nocache'].get('argmax_agreement'))" $1 $2; }
for r in 1 2; do for nf in 1 0; do
  TKV_NORM_FOLD=$nf timeout 900 python bench.py --no-cpu-baseline --nocache-queries 50 > gpurun_out/nf_c2_${nf}_$r.json 2>/dev/null; show gpurun_out/nf_c2_${nf}_$r.json c2_fold${nf}_run$r
done; done
TKV_NORM_FOLD=1 timeout 900 python bench.py --config c3 --queries 500 --capacity 256 --steps 2 --warmup 3 --nocache-queries 20 --no-cpu-baseline > gpurun_out/nf_c3_1.json 2>/dev/null; show gpurun_out/nf_c3_1.json c3_fold1
TKV_NORM_FOLD=0 timeout 900 python bench.py --config c3 --queries 500 --capacity 256 --steps 2 --warmup 3 --nocache-queries 20 --no-cpu-baseline > gpurun_out/nf_c3_0.json 2>/dev/null; show gpurun_out/nf_c3_0.json c3_fold0
