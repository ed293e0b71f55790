"""DRAM traffic per launch from `ncu --set full` raw CSV exports (ncu -i X.ncu-rep --page raw
--csv): writes profiles/<out>.json mapping kernel base name -> {dram_bytes, duration_us,
launches} (averaged over the captured launches).  bench.py reads it for roofline.traffic.

    python tools/ncu_traffic.py profiles/r1_traffic.json gpurun_out/prof_chol_raw.csv ...
"""
import csv
import json
import re
import sys


def base(name):
    name = re.sub(r"\(.*$", "", name)  # drop the argument list
    name = name.replace("unnamed>::", "").replace("(anonymous namespace)::", "").replace("tsvd::", "")
    return re.sub(r"^void ", "", name).split("<")[0].strip()


def main(out, files):
    acc = {}
    for f in files:
        rows = list(csv.reader(open(f)))
        hdr, units = rows[0], rows[1]
        ix = {k: hdr.index(k) for k in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                        "gpu__time_duration.sum")}
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e3, "us": 1.0, "ns": 1e-3}
        for r in rows[2:]:
            k = base(r[ix["Kernel Name"]])
            b = sum(float(r[ix[m]]) * scale[units[ix[m]]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            d = float(r[ix["gpu__time_duration.sum"]]) * scale[units[ix["gpu__time_duration.sum"]]]
            a = acc.setdefault(k, [0.0, 0.0, 0])
            a[0] += b
            a[1] += d
            a[2] += 1
    res = {k: {"dram_bytes": v[0] / v[2], "duration_us": v[1] / v[2], "launches": v[2],
               "src": "ncu --set full --clock-control none (dram__bytes_read.sum + dram__bytes_write.sum)"}
           for k, v in acc.items()}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
