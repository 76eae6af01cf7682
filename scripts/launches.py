"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        v = float(r[mi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        agg[r[ki].split("(")[0].replace("void ", "")].append(v)
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append((k, len(v), sum(v) / len(v), sum(v), sum(v) / tot))
    return out


if __name__ == "__main__":
    for k, n, avg, tot, share in summarise(sys.argv[1]):
        print(f"{k:36s} n={n:5d} avg={avg:9.2f}us total={tot:10.1f}us share={share * 100:5.1f}%")
