"""DRAM traffic per launch of the dominant kernels from ncu --set full reports.

usage: python tools/ncu_traffic.py OUT.json REPORT.ncu-rep [REPORT.ncu-rep ...]
Reads dram__bytes_read.sum + dram__bytes_write.sum and gpu__time_duration.sum
of every profiled launch (ncu -i ... --page raw --csv) and writes the per-kernel
averages that bench.py reports as roofline "traffic".
"""
import csv
import io
import json
import subprocess
import sys


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr = r[0]
    units = r[1]
    return hdr, units, r[2:]


def to_bytes(v, unit):
    v = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    if unit not in scale:
        raise ValueError(f"unknown byte unit {unit!r}")
    return v * scale[unit]


def to_ns(v, unit):
    v = float(v.replace(",", ""))
    scale = {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3,
             "ms": 1e6, "s": 1e9}
    if unit not in scale:
        raise ValueError(f"unknown time unit {unit!r}")
    return v * scale[unit]


def main():
    out, reps = sys.argv[1], sys.argv[2:]
    agg = {}
    for rep in reps:
        hdr, units, data = rows(rep)
        kn = hdr.index("Kernel Name")
        ir, iw, it = (hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum"),
                      hdr.index("gpu__time_duration.sum"))
        for r in data:
            name = r[kn].split("(")[0].split("::")[-1].split("<")[0].strip()
            if name.startswith("void "):
                name = name[5:]
            b = to_bytes(r[ir], units[ir]) + to_bytes(r[iw], units[iw])
            t = to_ns(r[it], units[it])
            a = agg.setdefault(name, {"launches": 0, "bytes": 0.0, "ns": 0.0, "reports": []})
            a["launches"] += 1
            a["bytes"] += b
            a["ns"] += t
            if rep not in a["reports"]:
                a["reports"].append(rep)
    res = {"note": "ncu --set full (cold cache, serialised replay): DRAM bytes per launch",
           "kernels": {k: {"launches": v["launches"],
                           "dram_bytes_per_launch": v["bytes"] / v["launches"],
                           "duration_ns_per_launch": v["ns"] / v["launches"],
                           "reports": v["reports"]} for k, v in agg.items()}}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
