"""Summarise ncu evidence into profiles/ (run here, on the CPU box, over
reports brought back from the B200 in gpurun_out/).

    python profiles/summarize.py --round r01 --launches gpurun_out/launches8.csv \
        --report gpurun_out/prof_jtj8.ncu-rep --config arap_warp [--report ... --config ...]

Writes profiles/<round>_launches.md (per-kernel device time shares from the
`gpu__time_duration.sum --clock-control none` launch list) and merges
per-kernel metrics into profiles/ncu_summary.json, which bench.py reads for
`roofline.traffic` (dram bytes read+write per launch of the J^T J p kernel).
"""
import argparse
import collections
import csv
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "lts__t_sector_hit_rate.pct", "launch__shared_mem_per_block_dynamic",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def launches(path, last=0):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    ni = hdr.index("Metric Name") if "Metric Name" in hdr else None
    agg = collections.defaultdict(list)
    body = [r for r in rows[hi + 1:] if len(r) > mi and (ni is None or r[ni] == "gpu__time_duration.sum")]
    if last:  # only the final `last` launches (one timed solve after the tuning launches)
        body = body[-last:]
    for r in body:
        v = float(r[mi].replace(",", "")) * UNIT.get(r[ui], 1.0) * 1e6  # -> us
        agg[r[ki].split("(")[0].replace("void ", "")].append(v)
    tot = sum(sum(v) for v in agg.values())
    return [(k, len(v), sum(v) / len(v), sum(v), sum(v) / tot) for k, v in
            sorted(agg.items(), key=lambda kv: -sum(kv[1]))]


def report_metrics(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                d[m] = v * UNIT.get(units[i], 1.0)
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--report", action="append", default=[])
    ap.add_argument("--config", action="append", default=[])
    ap.add_argument("--note", default="")
    ap.add_argument("--last", type=int, default=0, help="summarise only the final N launches")
    a = ap.parse_args()
    if a.launches:
        rows = launches(a.launches, a.last)
        with open(os.path.join(HERE, f"{a.round}_launches.md"), "w") as f:
            f.write(f"# {a.round}: ncu launch list ({os.path.basename(a.launches)})\n\n")
            f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` over the bench command; "
                    "cold-cache serialised launches, so compare SHARES, not absolutes.\n")
            if a.note:
                f.write(f"\n{a.note}\n")
            f.write("\n| kernel | launches | avg us | total us | share |\n|---|---|---|---|---|\n")
            for k, n, avg, tot, share in rows:
                f.write(f"| `{k}` | {n} | {avg:.2f} | {tot:.1f} | {share * 100:.1f}% |\n")
    summ_path = os.path.join(HERE, "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    for rep, cfg in zip(a.report, a.config):
        for d in report_metrics(rep):
            key = "jtj" if "jtj" in d["kernel"] else ("bm" if "_bm" in d["kernel"] else d["kernel"])
            rb = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
            d["dram_bytes"] = rb
            d["round"] = a.round
            d["report"] = os.path.basename(rep)
            summ.setdefault(cfg, {})[key] = d
    with open(summ_path, "w") as f:
        json.dump(summ, f, indent=1, sort_keys=True)
    print(open(os.path.join(HERE, f"{a.round}_launches.md")).read() if a.launches else "", file=sys.stderr)


if __name__ == "__main__":
    main()
