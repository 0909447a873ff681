"""Attribute ncu per-instruction counters to source lines.

usage: python profiles/sass_lines.py <ncu-rep> <kernel-mangled-name> <lib.so> [topN]
Joins `ncu --page source --print-source=sass` with `nvdisasm --print-line-info-inline`
of the same cubin (instruction i of the kernel <-> offset 16*i).
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kern, so = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
prefer = sys.argv[5] if len(sys.argv) > 5 else None  # attribute to first frame in this file
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) >= len(hdr)]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "--print-line-info-inline", os.path.join(tmp, cub)],
                     capture_output=True, text=True).stdout.splitlines()
start = None
for i, l in enumerate(dis):
    if l.startswith(f".text.{kern}:"):
        start = i
        break
cur = ("?", 0)
lines = {}
in_block = False
for l in dis[start + 1:]:
    if l.startswith("//---------------------") or l.startswith(".text."):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        loc = (os.path.basename(m.group(1)), int(m.group(2)))
        if not in_block:  # first line of a block = innermost inlined location
            cur = loc
            found = prefer is None or loc[0] == prefer
        elif not found and loc[0] == prefer:
            cur = loc
            found = True
        in_block = True
        continue
    in_block = False
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m:
        lines.setdefault(int(m.group(1), 16), cur)
instr = collections.Counter()
stall = collections.Counter()
tot_i = tot_s = 0
for k, r in enumerate(data):
    key = lines.get(16 * k, ("?", 0))
    n = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    instr[key] += n
    stall[key] += s
    tot_i += n
    tot_s += s
print(f"instructions {tot_i}  stall samples {tot_s}")
for key, n in instr.most_common(top):
    print(f"{key[0]:18s}:{key[1]:<5d} instr {100*n/tot_i:6.2f}%  stall {100*stall[key]/max(tot_s,1):6.2f}%")
