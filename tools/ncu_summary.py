"""Summarize an ncu report: key raw metrics per kernel and the top source
lines (stall samples) of a kernel.  Usage:
  python tools/ncu_summary.py REPORT.ncu-rep [kernel-regex] [n_lines]"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'launch__registers_per_thread', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'smsp__thread_inst_executed_per_inst_executed.ratio',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum']


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print("----", r[hdr.index("Kernel Name")][:60])
        for k in KEYS:
            if k in hdr:
                print(f"  {k:70s} {r[hdr.index(k)]} {units[hdr.index(k)]}")


def stalls(rep, kern, n):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur, hdr = None, None
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, ""])
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit():
            continue

        def f(x):
            try:
                return float(x)
            except ValueError:
                return 0.0
        a = agg[(cur, int(r[0]))]
        a[0] += f(r[hdr.index("Warp Stall Sampling (All Samples)")])
        a[1] += f(r[hdr.index("Instructions Executed")])
        a[2] += f(r[hdr.index("Thread Instructions Executed")])
        a[3] = r[1][:80].strip()
    ts = sum(v[0] for v in agg.values()) or 1
    te = sum(v[1] for v in agg.values()) or 1
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
        print(f"{k[0]:16s}:{k[1]:4d} samp {v[0] / ts * 100:5.1f}% inst {v[1] / te * 100:5.1f}% "
              f"lanes {v[2] / max(v[1], 1):5.1f} | {v[3]}")


if __name__ == "__main__":
    raw(sys.argv[1])
    if len(sys.argv) > 2:
        stalls(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
