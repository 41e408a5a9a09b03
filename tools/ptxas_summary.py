#!/usr/bin/env python
"""Registers and spills per sweep3d instantiation from the ptxas -v logs."""
import glob
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pat = sys.argv[1] if len(sys.argv) > 1 else "sweep3d"
for f in sorted(glob.glob(os.path.join(ROOT, "paper_1608_08658_b200/csrc/build/*.ptxas.log"))):
    name = None
    spill = ""
    for line in open(f):
        m = re.search(r"Compiling entry function '(\w+)'", line)
        if m:
            name = m.group(1)
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m:
            spill = f"spill {m.group(1)}/{m.group(2)}"
        m = re.search(r"Used (\d+) registers", line)
        if m and name and pat in name:
            dm = re.search(r"(sweep3d_\w*kernel)I(.*?)EEEv", name)
            short = (dm.group(1), re.findall(r"(?:Li|Lb|b)(\d+)", dm.group(2))) if dm else name
            print(short, "regs", m.group(1), spill)
            name = None
