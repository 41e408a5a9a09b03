#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel: launches, total / mean time and share of the GPU time.

  python tools/launch_list.py <launches.csv> "<command it profiled>" > launches.json
"""
import csv
import io
import json
import sys


def main(path, source):
    text = open(path).read()
    text = text[text.index('"ID"'):]  # skip ncu's own log lines
    rows = list(csv.DictReader(io.StringIO(text)))
    kern = {}
    total = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[r["Metric Unit"]]
        t = float(r["Metric Value"].replace(",", "")) * scale
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        e = kern.setdefault(name, {"launches": 0, "total_us": 0.0})
        e["launches"] += 1
        e["total_us"] += t
        total += t
    for e in kern.values():
        e["mean_us"] = e["total_us"] / e["launches"]
        e["share"] = e["total_us"] / total
    print(json.dumps({"source": source, "launches": sum(e["launches"] for e in kern.values()),
                      "total_us": total,
                      "kernels": dict(sorted(kern.items(), key=lambda kv: -kv[1]["total_us"]))},
                     indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
