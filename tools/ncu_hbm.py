"""Summarise an ncu CSV (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum)
per kernel: launches, device time, DRAM traffic and achieved DRAM bandwidth against the measured
HBM copy bandwidth (MEASURED_PEAKS.json hbm_gbs).

    python tools/ncu_hbm.py gpurun_out/hbm_c5.csv [out.txt]
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:  # pragma: no cover
    PEAK = 6541.1
UNITS = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
         "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main(path, out=None):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ii, ki, mi, vi, ui = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    per = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        per[r[ii]]["name"] = r[ki].split("(")[0].replace("void ", "").replace("tsvd::<unnamed>::", "")
        per[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * UNITS.get(r[ui], 1.0)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for x in per.values():
        a = agg[x["name"]]
        a[0] += 1
        a[1] += x.get("gpu__time_duration.sum", 0.0)
        a[2] += x.get("dram__bytes_read.sum", 0.0) + x.get("dram__bytes_write.sum", 0.0)
    lines = [f"DRAM bandwidth per kernel (ncu, serialised, cold L2 per replay); peak = {PEAK:.0f} GB/s measured copy",
             f"{'launches':>8} {'ms':>9} {'MB/launch':>10} {'GB/s':>8} {'frac':>6}  kernel"]
    for n, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        gbs = b / t / 1e9 if t else 0.0
        lines.append(f"{c:8d} {1e3 * t:9.3f} {b / c / 1e6:10.1f} {gbs:8.0f} {gbs / PEAK:6.2f}  {n[:90]}")
    txt = "\n".join(lines)
    print(txt)
    if out:
        open(out, "w").write(txt + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
