#!/bin/bash
# usage: profiles/stage_breakdown.sh <ncu-rep>   (per-engine-stage share of instructions/stalls)
REP=$1
python "$(dirname "$0")/sass_lines.py" "$REP" ${KNAME:-_Z14minhash_kernelILi22EEv11MinhashArgs} paper_2005_11547_b200/libdsk_b200.so 600 dsk_engine.cuh > /tmp/eng_lines.txt
python - "$(dirname "$0")/../paper_2005_11547_b200/csrc/dsk_engine.cuh" <<'PY'
import re, sys
src = open(sys.argv[1]).read().splitlines()
# map line -> enclosing engine function by scanning "__device__ ... name(" definitions
owner = {}
cur = "prologue"
for i, l in enumerate(src, 1):
    m = re.match(r"\s+__device__ (?:__forceinline__ )?[\w:<>]+\s+(\w+)\(", l)
    if m:
        cur = m.group(1)
    m2 = re.match(r"\s+__device__ Engine\(", l)
    if m2:
        cur = "Engine(ctor)"
    owner[i] = cur
agg = {}
for l in open("/tmp/eng_lines.txt"):
    m = re.match(r"(\S+)\s*:(\d+)\s+instr\s+([\d.]+)%\s+stall\s+([\d.]+)%", l)
    if not m:
        continue
    f, ln, i, s = m.group(1), int(m.group(2)), float(m.group(3)), float(m.group(4))
    key = owner.get(ln, f) if f == "dsk_engine.cuh" else f
    a = agg.setdefault(key, [0.0, 0.0])
    a[0] += i
    a[1] += s
print(open("/tmp/eng_lines.txt").readline().strip())
for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:22s} instr {v[0]:6.2f}%  stall {v[1]:6.2f}%")
PY
