# round 2: timed vs untimed executor on the same box (per-window ends); layered loads with host profile; exp2 emulation A/B
set -x
timeout 900 python scratch/e2e_gap.py > gpurun_out/e2e_gap.txt 2>&1
TKV_LAYERED_LOADS=1 TKV_HOST_PROFILE=1 timeout 900 python scratch/e2e_gap.py > gpurun_out/e2e_gap_layered.txt 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --nocache-queries 0"
TKV_LIB=paper_2601_08743_b200/lib/emu2/libtkv.so timeout 900 $B > gpurun_out/c4_emu2.json 2> gpurun_out/c4_emu2.err
TKV_LIB=paper_2601_08743_b200/lib/emu4/libtkv.so timeout 900 $B > gpurun_out/c4_emu4.json 2> gpurun_out/c4_emu4.err
timeout 900 $B > gpurun_out/c4_base.json 2> gpurun_out/c4_base.err
cat gpurun_out/e2e_gap.txt
