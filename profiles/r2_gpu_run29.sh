# round 2 (late): K-rotation batching A/B (rows per batch of hoisted shared loads: 1 = previous
# kernel, 4 = new default, 8) and the untraced no-rotation / no-exponential probes, C4 200 queries
set -x
B="python bench.py --config c4 --queries 200 --steps 2 --warmup 3 --nocache-queries 0 --no-cpu-baseline"
for v in rb4 rb1 rb8 norot noexp rb4b rb1b; do
  case $v in rb4|rb4b) L="";; rb1b) L="TKV_LIB=paper_2601_08743_b200/lib/rb1/libtkv.so";; *) L="TKV_LIB=paper_2601_08743_b200/lib/$v/libtkv.so";; esac
  env $L timeout 900 $B > gpurun_out/ab29_$v.json 2> gpurun_out/ab29_$v.err
  grep -o '"attention_ms_per_step": [0-9.]*' gpurun_out/ab29_$v.json
done
