# round 2 (late): L2 prefetch of the next attention item's Q tiles (default) vs none (nq), C2 / C4;
# then the attention / parity GPU tests on the default build
set -x
B="python bench.py --steps 3 --warmup 3 --nocache-queries 0 --no-cpu-baseline"
for cfg in c2 c4; do
  timeout 900 $B --config $cfg > gpurun_out/ab35_${cfg}_qpf.json 2> gpurun_out/ab35_${cfg}_qpf.err
  TKV_LIB=paper_2601_08743_b200/lib/nq/libtkv.so timeout 900 $B --config $cfg > gpurun_out/ab35_${cfg}_nq.json 2> gpurun_out/ab35_${cfg}_nq.err
done
timeout 1200 python -m pytest tests -m gpu -x -q -k "tcgen05 or bf16 or paged or parity or executor or encode" > gpurun_out/pytest35.log 2>&1; tail -1 gpurun_out/pytest35.log
