"""Aggregate an ncu source page (instructions executed, stall samples) by
enclosing function of this repo's CUDA sources.
  python tools/ncu_by_function.py REPORT.ncu-rep kernel-regex [n]"""
import collections
import csv
import io
import re
import subprocess
import sys


def franges(path):
    try:
        src = open(path).read().split("\n")
    except OSError:
        return None
    res, cur = [], "?"
    for line in src:
        m = re.match(r"^(?:template <[^>]*>\s*)?(?:TS_HD|__device__|__global__|inline|static)[^(]*?\b(\w+)\(", line)
        if m:
            cur = m.group(1)
        res.append(cur)
    return res


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main(rep, kern, n=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    cache, cur, hdr = {}, None, None
    inst, samp = collections.Counter(), collections.Counter()
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] in ("File Path", "File Name"):
            cur = r[1]
            cache.setdefault(cur, franges(cur))
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit():
            continue
        f = cache.get(cur)
        ln = int(r[0])
        name = cur.split("/")[-1] + ":" + (f[ln - 1] if f and ln <= len(f) else "?")
        inst[name] += num(r[hdr.index("Instructions Executed")])
        samp[name] += num(r[hdr.index("Warp Stall Sampling (All Samples)")])
    ti, ts = sum(inst.values()) or 1, sum(samp.values()) or 1
    for k, v in inst.most_common(n):
        print(f"{k:50s} inst {v / ti * 100:5.1f}%  samples {samp[k] / ts * 100:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
