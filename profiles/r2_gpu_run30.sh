# round 2 (late): single-stream attention items (an item whose tokens fit the first Q tile runs
# stream 0 alone) — GPU suite, then C4 / C2 A/B against both streams on every item (ss0)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest30.log
B="python bench.py --steps 2 --warmup 3 --nocache-queries 0 --no-cpu-baseline"
for cfg in c4 c2; do
  for v in ss1 ss0; do
    if [ $v = ss1 ]; then L=""; else L="TKV_LIB=paper_2601_08743_b200/lib/ss0/libtkv.so"; fi
    env $L timeout 900 $B --config $cfg > gpurun_out/ab30_${cfg}_$v.json 2> gpurun_out/ab30_${cfg}_$v.err
  done
done
cat gpurun_out/pytest30.log
