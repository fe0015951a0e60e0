# executor host lead bound (TKV_HOST_LEAD) A/B on C3 and C2: value (timed kernels) and e2e (untimed)
set -u
timeout 900 python -m pytest tests/test_gpu.py -q -m gpu -k "executor or serving_path or edge" 2>&1 | tail -1
for c in "--config c3 --queries 500 --capacity 256 --steps 2" "--steps 3"; do for L in 2 0 3; do
  TKV_HOST_LEAD=$L timeout 900 python bench.py $c --warmup 3 --nocache-queries 0 --no-cpu-baseline > gpurun_out/hl.json 2>/dev/null
  python -c "import json,sys;d=json.load(open('gpurun_out/hl.json'));print(sys.argv[1],sys.argv[2],round(d['value'],1),round(d['ms_per_step'],1),round(d['e2e']['value'],1),d['e2e']['steps_call_makespan_serve_ms'][-1])" "$c" lead$L
done; done
