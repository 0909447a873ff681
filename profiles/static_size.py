"""Static SASS size of a kernel attributed to engine functions (innermost
dsk_engine.cuh frame).  usage: static_size.py <lib.so> <mangled kernel>"""
import collections, os, re, subprocess, sys, tempfile
so, kern = sys.argv[1], sys.argv[2]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "--print-line-info-inline", os.path.join(tmp, cub)],
                     capture_output=True, text=True).stdout.splitlines()
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..",
                        "paper_2005_11547_b200", "csrc", "dsk_engine.cuh")).read().splitlines()
owner, cur = {}, "top"
for i, l in enumerate(src, 1):
    m = re.match(r"\s+(?:template <[^>]*>\s*)?__device__ (?:__forceinline__ )?[\w:<>]+\s+(\w+)\(", l)
    if m:
        cur = m.group(1)
    owner[i] = cur
start = next(i for i, l in enumerate(dis) if l.startswith(f".text.{kern}:"))
counts = collections.Counter()
loc, found, in_block = ("?", 0), False, False
for l in dis[start + 1:]:
    if l.startswith("//---------------------"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        f = (os.path.basename(m.group(1)), int(m.group(2)))
        if not in_block:
            loc, found = f, f[0] == "dsk_engine.cuh"
        elif not found and f[0] == "dsk_engine.cuh":
            loc, found = f, True
        in_block = True
        continue
    in_block = False
    if re.search(r"/\*[0-9a-f]{4,}\*/", l):
        key = owner.get(loc[1], "?") if loc[0] == "dsk_engine.cuh" else loc[0]
        counts[key] += 1
tot = sum(counts.values())
print(f"total {tot} instr = {tot*16/1024:.0f} KB")
for k, v in counts.most_common(25):
    print(f"{k:24s} {v:6d}  {v*16/1024:6.1f} KB")
