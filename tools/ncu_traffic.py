"""DRAM traffic of a kernel class from an ncu launch list taken over ONE update
(`ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv ... python tools/profile_one.py <cfg>`): the class's DRAM bytes per
launch (the sum over its kernels — for the DMMA GEMM class the GEMM and split-K reduce kernels —
divided by their count), written to profiles/r2_traffic_<cfg>.json for bench.py's
roofline.traffic.  bench.py puts it beside the algorithmic bytes per launch the library
accounts for the same class over the same kind of update, so the two compare like with like.

    python tools/ncu_traffic.py c4 gpurun_out/traffic_c4.csv
"""
import collections
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLASSES = {"dgemm_dmma": r"dgemm_v2_kernel|dgemm_kernel|splitk_reduce|items_reduce|kr_plan"}
UNITS = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(cfg, path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ii, ki, mi, vi, ui = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    per = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            per[r[ii]]["name"] = r[ki]
            per[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * UNITS.get(r[ui], 1.0)
    out = {}
    for cls, rx in CLASSES.items():
        ks = [x for x in per.values() if re.search(rx, x["name"])]
        if not ks:
            continue
        b = sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in ks)
        t = sum(x.get("gpu__time_duration.sum", 0) for x in ks)
        out[cls] = {"dram_bytes": b / len(ks), "launches": len(ks), "ms": 1e3 * t,
                    "what": f"ncu over one {cfg} update (tools/profile_one.py): mean DRAM read+write bytes per launch "
                            f"of the {len(ks)} launches of the class"}
    dst = os.path.join(ROOT, "profiles", f"r2_traffic_{cfg}.json")
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
