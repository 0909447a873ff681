import csv, io, subprocess, sys, collections, re
rep=sys.argv[1]
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
rows=list(csv.reader(io.StringIO(sass)))
hdr=rows[1]; ix={h:i for i,h in enumerate(hdr)}
#print(hdr)
src=[k for k in hdr if k.lower().startswith('source')][0]
ie=[k for k in hdr if 'Instructions Executed' in k and 'Thread' not in k][0]
c=collections.Counter(); tot=0
special=collections.Counter()
for r in rows[2:]:
    if len(r)<len(hdr): continue
    t=r[ix[src]].strip()
    try: n=float(r[ix[ie]])
    except: continue
    m=re.match(r'(@!?U?P\d+\s+)?([A-Z0-9_]+)',t)
    op=m.group(2) if m else '?'
    c[op]+=n; tot+=n
    if 'SR_CgaCtaId' in t: special['S2R CgaCtaId']+=n
    if 'LDL' in t or 'STL' in t: special['local']+=n
for op,n in c.most_common(32): print(f"{op:12s} {n/tot*100:6.2f}%")
for k,v in special.items(): print(k, f"{v/tot*100:.2f}%")
