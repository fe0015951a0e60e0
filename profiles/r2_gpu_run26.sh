# round 2: bf16 oracle mirrors the RMSNorm fold — Llama-width parity report; then the GEMM variants at C4/C5
set -x
TKV_PARITY_REPORT=gpurun_out/parity_fold.json timeout 1500 python -m pytest tests -m gpu -x -q -k "parity or bf16 or paged or fold" 2>&1 | tail -5 > gpurun_out/gpu_parity26.log
bash profiles/r2_gpu_run24.sh
cat gpurun_out/gpu_parity26.log
