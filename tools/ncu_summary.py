"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.

    python tools/ncu_summary.py gpurun_out/launches.csv [out.txt]
ncu times are cold-cache and serialised: compare SHARES, not absolutes."""
import collections
import csv
import sys


def summarize(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(r[ui], 1e-6)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = [f"launches {sum(v[0] for v in agg.values())}  total {tot:.2f} ms (ncu, cold-cache, serialised)",
             f"{'ms':>10} {'share':>6} {'launches':>8} {'us/launch':>10}  kernel"]
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{t:10.2f} {100 * t / tot:5.1f}% {c:8d} {1e3 * t / c:10.1f}  {n}")
    return "\n".join(lines)


if __name__ == "__main__":
    out = summarize(sys.argv[1])
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(out + "\n")
    print(out)
