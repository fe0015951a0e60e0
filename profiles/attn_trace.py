#!/usr/bin/env python3
"""Print CTA 0's timeline from a TKV_ATTN_TRACE dump of attn_tc5_kernel (debug instrumentation):
per K/V tile g the ns offsets of TMA issue, MMA acquire/commit, softmax S-ready / P-ready."""
import sys

import numpy as np

t = np.fromfile(sys.argv[1], np.uint32).reshape(-1, 1024).astype(np.int64)
t0 = t[10, 0]
rel = lambda x: (x - t0) if x else -1
names = ["K_issue", "V_issue", "mma_kfull", "QK_commit", "mma_pfull", "sm_sfull", "sm_pready", "", "", "K_ready", "",
         "mma_vfull", "sm_sload", "sm_max", "sm_exp", "sm1_pready", "pv0_issued", "pv1_issued", "mma_pfull1",
         "qk0_issued", "sm1_sfull", "sm1_exp"]
print("items: Q issue / epilogue done")
for j in range(1024):
    if not t[8, j]:
        break
    print("  j=%d  %8d %8d" % (j, rel(t[8, j]), rel(t[7, j])))
cols = [c for c in [0, 9, 1, 11, 2, 19, 5, 12, 13, 14, 6, 4, 16, 20, 21, 15, 18, 17, 3] if c < t.shape[0]]
print("g     " + " ".join("%10s" % names[c] for c in cols))
for g in range(1024):
    if not t[0, g]:
        break
    print("%4d  " % g + " ".join("%10d" % rel(t[c, g]) for c in cols))
