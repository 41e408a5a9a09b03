#!/usr/bin/env python
"""Static SASS mix of one sweep kernel instantiation, split at the consumer's
full-barrier waits (one chunk per unrolled plane phase)."""
import collections
import re
import subprocess
import sys

so = "paper_1608_08658_b200/libsfdb200.so"
pat = sys.argv[1]  # e.g. sweep3d_kernelILi4ELi4ELi2ELi3ELb0ELb1E
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    lines = [l for l in f.split("\n") if re.match(r"\s*/\*[0-9a-f]{4,}\*/", l)]
    ops = []
    for l in lines:
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", l)
        if m:
            ops.append(m.group(2))
    print(name[:100], "static instructions:", len(ops))
    c = collections.Counter(ops)
    print(c.most_common(30))
    break
