"""Split ncu source-page warp-stall samples into barrier waits and everything
else ("work": what the warps that are not waiting at a CTA barrier do), per
source line.  In a CTA-cooperative engine the work lines are the critical
path; the barrier lines only say where the other warps wait for it.

  ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > x.csv
  python tools/ncu_source_work.py x.csv [top]
"""
import collections
import csv
import sys

cur = None
hdr = None
work = collections.Counter()
wait = collections.Counter()
reason = collections.defaultdict(collections.Counter)
seen = set()
last = None
for r in csv.reader(open(sys.argv[1])):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        i_all = r.index("Warp Stall Sampling (All Samples)")
        i_bar = r.index("stall_barrier")
        stall_cols = [(i, n) for i, n in enumerate(r) if n.startswith("stall_") and "Not Issued" not in n]
        continue
    if hdr is None or len(r) <= i_bar:
        continue
    if r[0]:
        last = r[0]
    if not r[2] or r[2] in seen:
        continue
    seen.add(r[2])
    try:
        tot = float(r[i_all] or 0)
        bar = float(r[i_bar] or 0)
    except ValueError:
        continue
    key = (cur, last)
    wait[key] += bar
    work[key] += tot - bar
    for i, n in stall_cols:
        if n != "stall_barrier":
            try:
                reason[key][n] += float(r[i] or 0)
            except ValueError:
                pass
top = int(sys.argv[2]) if len(sys.argv) > 2 else 50
tw, tb = sum(work.values()), sum(wait.values())
print(f"samples: work {tw:.0f} ({100 * tw / (tw + tb):.1f} %), barrier wait {tb:.0f}")
print("-- work lines (share of work samples; top reasons)")
for key, s in work.most_common(top):
    rs = ", ".join(f"{n[6:]} {100 * v / max(s, 1):.0f}%" for n, v in reason[key].most_common(3))
    print(f"{100 * s / tw:5.2f}% {key[0]}:{key[1]}   [{rs}]")
print("-- barrier-wait lines (share of barrier samples)")
for key, s in wait.most_common(25):
    print(f"{100 * s / tb:5.2f}% {key[0]}:{key[1]}")
