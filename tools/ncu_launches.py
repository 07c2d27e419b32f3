"""Per-kernel averages from an `ncu --metrics ... --csv` launch list
(gpu__time_duration.sum and, when captured, dram bytes)."""
import collections
import csv
import io
import sys


def main(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    hdr = rows[0]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = collections.defaultdict(dict)
    for r in rows[1:]:
        if len(r) == len(hdr):
            d[(int(r[ii]), r[ki][:70])][r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.defaultdict(list)
    for (_, k), m in sorted(d.items()):
        agg[k].append(m)
    for k, ms in agg.items():
        n = len(ms)
        avg = lambda key: sum(m.get(key, 0.0) for m in ms) / n
        print(f"{k:70s} n={n:3d} avg={avg('gpu__time_duration.sum') / 1e3:9.1f} us "
              f"rd={avg('dram__bytes_read.sum') / 1e6:8.1f} MB wr={avg('dram__bytes_write.sum') / 1e6:8.1f} MB")


if __name__ == "__main__":
    main(sys.argv[1])
