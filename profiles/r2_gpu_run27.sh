# round 2 (late): MUFU ex2 rate microbenchmark; C4 attention CTA-0 timelines with the MMA issue
# points traced (baseline, no K rotation, no exponentials) to find what paces the tile period
set -x
./scratch/ex2_bench > gpurun_out/ex2_bench.txt 2>&1
B="python bench.py --config c4 --queries 200 --steps 1 --warmup 3 --nocache-queries 0 --no-cpu-baseline"
for v in base norot noexp; do
  if [ $v = base ]; then L=""; else L="TKV_LIB=paper_2601_08743_b200/lib/$v/libtkv.so"; fi
  env $L TKV_ATTN_TRACE=gpurun_out/attn_$v.bin timeout 900 $B > gpurun_out/attn_$v.json 2> gpurun_out/attn_$v.err
  python profiles/attn_trace.py gpurun_out/attn_$v.bin > gpurun_out/attn_$v.txt 2>&1
done
cat gpurun_out/ex2_bench.txt
