"""Static SASS instruction count per engine function (innermost engine frame).

usage: python profiles/static_fn.py <sass-with-line-info>   (nvdisasm --print-line-info-inline)
"""
import collections
import re
import sys

src = open("paper_2005_11547_b200/csrc/dsk_engine.cuh").read().splitlines()
fn, cur_fn = {}, "helpers"
for i, l in enumerate(src, 1):
    m = re.match(r"\s+(?:template <[^>]*>\s*)?__device__ (?:__forceinline__ |__noinline__ )?[\w:<>]+\s+(\w+)\(", l)
    if m:
        cur_fn = m.group(1)
    if re.match(r"\s+__device__ Engine\(", l):
        cur_fn = "ctor"
    fn[i] = cur_fn
cnt = collections.Counter()
chain, fresh = [], False
for l in open(sys.argv[1]):
    if "//##" in l:
        if not fresh:  # a new location block starts after an instruction
            chain, fresh = [], True
        chain += re.findall(r'"([^"]+)", line (\d+)', l)
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+[A-Z@]", l):
        tag = None
        for f, n in chain:
            if f.endswith("dsk_engine.cuh"):
                tag = fn.get(int(n), "?")
                break
        if tag is None:
            tag = chain[0][0].split("/")[-1] if chain else "?"
        cnt[tag] += 1
        fresh = False
for k, v in cnt.most_common(40):
    print(f"{k:24s} {v}")
