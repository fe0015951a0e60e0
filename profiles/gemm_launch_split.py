#!/usr/bin/env python3
"""Per-projection GEMM times from an ncu launch list of one serving step (bench.py under
TKV_NCU=1): the GEMM launches of a window are [qkv, o, gate/up, down] x layers + head."""
import csv
import statistics
import sys


def main(fn, layers=32):
    rows = list(csv.reader(open(fn)))
    hdr, g = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum" and "gemm" in d["Kernel Name"]:
                g.append(float(d["Metric Value"].replace(",", "")) / 1e3)
    per = {k: [] for k in ("qkv", "o", "gate_up", "down", "head")}
    names = ["qkv", "o", "gate_up", "down"]
    for i, t in enumerate(g):
        k = i % (4 * layers + 1)
        per["head" if k == 4 * layers else names[k % 4]].append(t)
    for k, v in per.items():
        if v:
            print("%-8s n=%4d mean %7.1f us  total %8.1f ms" % (k, len(v), statistics.mean(v), sum(v) / 1e3))


if __name__ == "__main__":
    main(sys.argv[1])
