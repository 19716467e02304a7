"""Turn the ncu metrics CSV of tools/gpu_ncu.sh (one ttgbf_filter_run launch,
application replay) into the DRAM-traffic record bench.py reads
(profiles/rNN_ncu_dram_c5.json).

  python tools/ncu_dram_json.py metrics.csv prof_run.log out.json
"""
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
iname, ival = hdr.index("Metric Name"), hdr.index("Metric Value")
m = {}
for r in rows[1:]:
    try:
        m[r[iname]] = float(r[ival].replace(",", ""))
    except ValueError:
        pass
att = None
for line in open(sys.argv[2]):
    line = line.strip()
    if line.startswith("{") and "attempted" in line:
        att = json.loads(line)["attempted"]
rd, wr = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
rec = {
    "command": "tools/gpu_ncu.sh: ncu --replay-mode application --profile-from-start off --clock-control none "
               "--metrics ... python tools/prof_run.py --batch 296 --warmup 2 --steps 1",
    "kernel": f"ttgbf_filter_run ({att} filters x 1 attempted step, C5 workload)",
    "dram_bytes_read": rd, "dram_bytes_write": wr, "duration_ns": m.get("gpu__time_duration.sum"),
    "l2_hit_pct": m.get("lts__t_sector_hit_rate.pct"), "l1_hit_pct": m.get("l1tex__t_sector_hit_rate.pct"),
    "l2_bytes": m.get("lts__t_bytes.sum"),
    "attempted_steps": att, "dram_bytes_per_attempted_step": (rd + wr) / att,
    "metrics": m,
}
json.dump(rec, open(sys.argv[3], "w"), indent=1)
print(json.dumps({k: rec[k] for k in ("dram_bytes_per_attempted_step", "l2_hit_pct", "l1_hit_pct", "duration_ns")}))
