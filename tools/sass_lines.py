#!/usr/bin/env python
"""SASS instruction count per source line for one kernel of a cubin (needs -lineinfo).
Usage: python tools/sass_lines.py file.cubin kernel-substring [N]"""
import collections
import re
import subprocess
import sys

cubin, target = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
cnt, infn, line = collections.Counter(), False, None
for l in out.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        infn = target in m.group(1)
        continue
    if not infn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        line = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        cnt[line] += 1
byfile = collections.Counter()
for (f, _), c in cnt.items():
    byfile[f] += c
print("total", sum(cnt.values()), byfile.most_common(8))
for k, c in cnt.most_common(n):
    print(c, k)
