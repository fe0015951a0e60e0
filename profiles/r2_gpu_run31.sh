# round 2 (late): P published in two halves (PV's first four k-steps overlap the softmax's second
# half; TKV_ATTN_PHALF=1 build) — attention / parity tests on that build, then C4 / C5 A/B
set -x
L=paper_2601_08743_b200/lib/ph/libtkv.so
TKV_LIB=$L timeout 1200 python -m pytest tests -m gpu -x -q -k "tcgen05 or bf16 or paged or parity or executor" 2>&1 | tail -5 > gpurun_out/pytest31_ph.log
B="python bench.py --steps 2 --warmup 3 --nocache-queries 0 --no-cpu-baseline"
TKV_LIB=$L timeout 900 $B --config c4 > gpurun_out/ab31_c4_ph.json 2> gpurun_out/ab31_c4_ph.err
timeout 900 $B --config c4 > gpurun_out/ab31_c4_base.json 2> gpurun_out/ab31_c4_base.err
TKV_LIB=$L timeout 1200 $B --config c5 > gpurun_out/ab31_c5_ph.json 2> gpurun_out/ab31_c5_ph.err
timeout 1200 $B --config c5 > gpurun_out/ab31_c5_base.json 2> gpurun_out/ab31_c5_base.err
cat gpurun_out/pytest31_ph.log
