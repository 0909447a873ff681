"""Print the SASS of one kernel with per-instruction execution counts and the
source line (innermost inlined frame) each instruction comes from.

usage: python profiles/sass_dump.py <ncu-rep> <kernel-mangled-name> <lib.so> [file:lo-hi ...]
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kern, so = sys.argv[1], sys.argv[2], sys.argv[3]
ranges = []
for a in sys.argv[4:]:
    f, r = a.split(":")
    lo, hi = (int(x) for x in r.split("-"))
    ranges.append((f, lo, hi))
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
start = next(i for i, l in enumerate(dis) if l.startswith(f".text.{kern}:"))
cur = ("?", 0)
lines = {}
in_block = False
for l in dis[start + 1:]:
    if l.startswith(".text."):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        if not in_block:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
        in_block = True
        continue
    in_block = False
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m:
        lines.setdefault(int(m.group(1), 16), cur)
src_col = ix.get("Source", 1)
for k, r in enumerate(data):
    key = lines.get(16 * k, ("?", 0))
    if ranges and not any(key[0] == f and lo <= key[1] <= hi for f, lo, hi in ranges):
        continue
    n = int(r[ix["Instructions Executed"]] or 0)
    if n == 0:
        continue
    print(f"{16*k:06x} {n:12d} {key[0]}:{key[1]:<4d} {r[src_col].strip()}")
