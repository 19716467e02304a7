"""Aggregate ncu --page source --print-source cuda,sass CSV exports by source line
(warp-stall samples, each SASS address counted once).

  ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > x.csv
  python tools/ncu_source_agg.py x.csv [top]
"""
import csv, collections, sys
cur_file=None; agg=collections.Counter(); seen=set(); last_line=None
hdr=None
rows=list(csv.reader(open(sys.argv[1])))
for r in rows:
    if not r: continue
    if r[0]=="File Path": cur_file=r[1].split('/')[-1]; continue
    if r[0]=="Function Name": continue
    if r[0]=="Line No": hdr=r; i_s=r.index("Warp Stall Sampling (All Samples)"); continue
    if hdr is None or len(r)<=i_s: continue
    if r[0]: last_line=r[0]
    addr=r[2]
    if not addr: continue
    try: s=float(r[i_s] or 0)
    except: continue
    key=(addr)
    if key in seen: continue
    seen.add(key)
    agg[(cur_file,last_line)]+=s
tot=sum(agg.values())
print("tot",tot)
for (f,l),s in agg.most_common(int(sys.argv[2]) if len(sys.argv)>2 else 70):
    print(f"{100*s/tot:5.2f}% {f}:{l}")
