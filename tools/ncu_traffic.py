#!/usr/bin/env python
"""Record the DRAM traffic per launch of one ncu --set full capture in
profiles/ncu_summary.json under the key bench.py looks up:
"<workload>|<instantiation>|z<zchunks>" (bench.ncu_traffic).

  python tools/ncu_traffic.py <report.ncu-rep> <bench line .json> <source path>

The bench line names the workload (config.workload's "<name>:" prefix), the
instantiation and z chunks it autotuned to (config.sweep); the capture must
have been taken with that tiling forced (SFDB200_TILE / SFDB200_ZCHUNKS), and
its kernel name must carry the same template arguments, else nothing is
written."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rep, line_path, source):
    line = json.loads(open(line_path).read().strip().splitlines()[-1])
    sweep = line["config"]["sweep"]
    name = line["config"]["workload"].split(":")[0]
    inst, zc = sweep["instantiation"], sweep["zchunks"]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    got = None
    for r in rows[2:]:
        kern = r[hdr.index("Kernel Name")]
        if kern.split("(")[0].replace("void ", "").strip() == inst:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = float(r[hdr.index("dram__bytes_read.sum")]) * scale[units[hdr.index("dram__bytes_read.sum")]]
            wr = float(r[hdr.index("dram__bytes_write.sum")]) * scale[units[hdr.index("dram__bytes_write.sum")]]
            got = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                   "kernel": kern[:120], "source": source}
            break
    if got is None:
        sys.exit(f"no launch of {inst} in {rep}")
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        d = json.load(open(p))
    except Exception:
        d = {}
    key = f"{name}|{inst}|z{zc}" + ("|dyn" if sweep.get("ctas") == -2 else "")
    d.setdefault("captures", {})[key] = got
    d["_key"] = "<workload>|<kernel instantiation>|z<zchunks> (bench.py ncu_traffic)"
    json.dump(d, open(p, "w"), indent=1)
    print(json.dumps(got))


if __name__ == "__main__":
    main(*sys.argv[1:4])
