"""Per-kernel summary of the last N launches of an ncu launch list with
gpu__time_duration + dram bytes:  python scripts/exp/ll_summary.py file.csv [N]"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 60
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
iK, iM, iV, iID = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per, names = collections.defaultdict(dict), {}
for r in rows[hi + 1:]:
    per[int(r[iID])][r[iM]] = float(r[iV].replace(",", ""))
    names[int(r[iID])] = r[iK]
agg, tot = collections.OrderedDict(), 0.0
for i in sorted(per)[-N:]:
    n = names[i].split("(")[0].split("<")[0].replace("void ", "")
    t = per[i].get("gpu__time_duration.sum", 0)
    b = per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0)
    a = agg.setdefault(n, [0, 0.0, 0.0])
    a[0] += 1; a[1] += t; a[2] += b
    tot += t
for n, (c, t, b) in agg.items():
    print(f"{n:28s} n={c:3d} total={t / 1e3:9.1f}us avg={t / c / 1e3:8.1f}us dram/launch={b / c / 1e9:6.3f}GB "
          f"{b / t if t else 0:6.2f} TB/s")
print("sum ms", tot / 1e6)
