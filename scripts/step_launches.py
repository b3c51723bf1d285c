"""Print the per-kernel launch list of the LAST step of an ncu
--metrics gpu__time_duration.sum,launch__grid_size CSV (scripts/profile_step.py
run with --steps 2), in launch order."""
import csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = {}
for r in rows[hi + 1:]:
    if len(r) > vi:
        d.setdefault(int(r[ii]), {"k": r[ki]})[r[mi]] = r[vi]
items = sorted(d.items())
last = items[len(items) // 2:]
tot = 0.0
for i, v in last:
    k = re.sub(r"\(.*", "", v["k"]).replace("dlrm::(anonymous namespace)::", "").replace("void ", "")
    t = float(v["gpu__time_duration.sum"].replace(",", "")) / 1e3
    tot += t
    print(f"{i:4d} {k[:60]:60s} {t:7.1f} us  grid={v.get('launch__grid_size')}")
print(f"total {tot:.1f} us over {len(last)} launches")
