"""Summarise an ncu metrics CSV of the GEMM launches of one factorization into
profiles/r02_ncu_gemm_traffic.json (read by bench.py for roofline.traffic).

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none -k regex:"k_gemm|k_rankk" --launch-skip 1 --csv \
        --log-file gpurun_out/ncu_gemm.csv python tools/one_factorization.py 5 32768
    python tools/ncu_traffic.py gpurun_out/ncu_gemm.csv profiles/r02_ncu_gemm_traffic.json

(--launch-skip 1 drops the input generator's GEMM, the first matching launch.)
"""
import csv
import io
import json
import sys
from collections import defaultdict


def main(src, dst):
    lines = [l for l in open(src) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    by = defaultdict(dict)
    for r in rows:
        v = float(r["Metric Value"].replace(",", ""))
        v *= {"us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "Kbyte": 1e3, "Mbyte": 1e6,
              "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(r["Metric Unit"], 1.0)
        by[r["ID"]][r["Metric Name"]] = v
        by[r["ID"]]["name"] = r["Kernel Name"].split("(")[0].split("::")[-1]
        by[r["ID"]]["grid"] = r["Grid Size"]
    per_kernel = defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "ns": 0.0})
    launches = []
    for i, d in by.items():
        b = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        k = per_kernel[d["name"]]
        k["launches"] += 1
        k["dram_bytes"] += b
        k["ns"] += d["gpu__time_duration.sum"]
        launches.append((d["gpu__time_duration.sum"], b, d["dram__bytes_read.sum"],
                         d["dram__bytes_write.sum"], d["name"], d["grid"]))
    launches.sort(reverse=True)
    top = launches[0]
    total = sum(l[1] for l in launches)
    out = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                     "gpu__time_duration.sum --clock-control none over the GEMM launches of one "
                     f"config-5 factorization (n=32768); {src}",
           "launches": len(launches), "dram_bytes_total": total,
           "dram_bytes_per_launch": total / max(len(launches), 1),
           "per_kernel": dict(per_kernel),
           "top_launch": {"kernel": top[4], "grid": top[5], "ncu_ms": top[0] / 1e6,
                          "dram_bytes": top[1], "dram_read": top[2], "dram_write": top[3]}}
    with open(dst, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
