"""Count local-memory spill instructions (STL/LDL) of one kernel per source
file (innermost inlined frame): python profiles/spills.py <lib.so> <kernel> [file]"""
import collections, os, re, subprocess, sys, tempfile
so, kern = sys.argv[1], sys.argv[2]
only = sys.argv[3] if len(sys.argv) > 3 else None
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "--print-line-info-inline", os.path.join(tmp, cub)],
                     capture_output=True, text=True).stdout.splitlines()
st = next(i for i, l in enumerate(dis) if l.startswith(f".text.{kern}:"))
cur, inb = ("?", 0), False
cnt = collections.Counter()
for l in dis[st + 1:]:
    if l.startswith(".text."):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        if not inb:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
        inb = True
        continue
    inb = False
    m = re.search(r"\b(STL|LDL)\b", l)
    if m and (only is None or cur[0] == only):
        cnt[(m.group(1), cur[0])] += 1
        if only:
            cnt[(m.group(1), cur)] += 1
for k, v in sorted(cnt.items(), key=str):
    print(k, v)
