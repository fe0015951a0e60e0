#!/usr/bin/env python3
"""Summarise ncu evidence for profiles/: per-kernel launch shares from a
`--metrics gpu__time_duration.sum --csv` launch list, and the key counters of `--set full`
captures (time, DRAM bytes, tensor-pipe and DRAM utilisation, registers, occupancy).

    python profiles/ncu_summary.py launches <launches.csv>
    python profiles/ncu_summary.py report <x.ncu-rep>
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_pct"),
    ("sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", "bf16_mma_ops_pct"),
    ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", "tcgen05_bf16_ops_pct"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_active_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__cycles_active.avg.pct_of_peak_sustained_elapsed", "smsp_active_pct"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "ID")
    data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0] != "ID"]
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"].replace(",", "")) * scale.get(d.get("Metric Unit", "nsecond"), 1.0)
    tot = sum(v[1] for v in agg.values())
    print("%-58s %6s %12s %7s" % ("kernel", "n", "total ms", "share"))
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print("%-58s %6d %12.3f %6.1f%%" % (k[:58], n, t / 1e6, 100 * t / tot))
    print("total %.3f ms over %d launches (cold-cache, serialised: compare shares)" % (tot / 1e6,
                                                                                   sum(v[0] for v in agg.values())))


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")][:70]
        print("== %s" % name)
        for key, short in KEYS:
            if key in hdr:
                i = hdr.index(key)
                print("   %-18s %s %s" % (short, r[i], units[i]))


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])
