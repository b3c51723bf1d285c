"""Warp-stall samples per CUDA source line from an `ncu --page source --csv
--print-source cuda,sass` dump: python scripts/ncu_lines.py dump.csv [n]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur, hdr, agg = None, None, {}
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5 or not r[0].isdigit():
        continue
    try:
        v = float(r[4]) if r[4] else 0.0
    except ValueError:
        v = 0.0
    k = (cur, int(r[0]))
    agg.setdefault(k, [0.0, r[1]])
    agg[k][0] += v
tot = sum(v[0] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
    print(f"{v[0] / tot * 100:5.1f}%", k, v[1].strip()[:100])
