#!/usr/bin/env python3
"""tcgen05 GEMM sweep on the serving shapes (one b_c=100 window of the c2 workload, Llama-3-8B
widths): TFLOP/s of the product kernel (persistent) vs the one-tile-per-CTA kernel, CUDA-event
timed (5 reps after a warm-up), plus a correctness check against numpy. Prints one JSON line."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_08743_b200 import native as N  # noqa: E402

SHAPES = [  # (name, M, N, K)
    ("qkv", 4992, 6144, 4096), ("o", 4992, 4096, 4096), ("gate_up", 4992, 28672, 4096),
    ("down", 4992, 4096, 14336), ("head", 100, 128256, 4096), ("qkv_small_m", 47, 6144, 4096),
]


def bits(x):
    return (x.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)


def main():
    rng = np.random.default_rng(0)
    out = {}
    for name, M, Nn, K in SHAPES:
        A = bits(rng.standard_normal((M, K)).astype(np.float32))
        B = bits((rng.standard_normal((Nn, K)) / np.sqrt(K)).astype(np.float32))
        res = {}
        for label, mode in (("persistent", 0), ("classic", 2)):
            c, ms = N.debug_gemm(A, B, epilogue=0, simt=mode)
            res[label + "_tflops"] = 2.0 * M * Nn * K / (ms * 1e-3) / 1e12
            res[label + "_ms"] = ms
        if M * Nn <= 4992 * 6144:
            ref = (A.astype(np.uint32) << 16).view(np.float32).astype(np.float64) @ \
                  (B.astype(np.uint32) << 16).view(np.float32).astype(np.float64).T
            got = (c.astype(np.uint32) << 16).view(np.float32)
            res["max_rel_err"] = float(np.abs(got - ref).max() / np.abs(ref).max())
        out[name] = res
    print(json.dumps(out))


if __name__ == "__main__":
    main()
