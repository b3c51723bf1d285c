"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel time of
the LAST step (launches after the first `--skip`), grouped by kernel name."""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
ids = hdr.index("ID")
recs = [(int(r[ids]), r[ki], float(r[vi].replace(",", ""))) for r in rows[hdr_i + 1:] if len(r) > vi]
n = len(recs)
half = recs[n // 2:] if len(sys.argv) < 3 else recs[int(sys.argv[2]):]
def short(k):
    k = re.sub(r"\(.*", "", k)
    k = k.replace("dlrm::(anonymous namespace)::", "").replace("void ", "")
    return k[:70]
agg = collections.OrderedDict()
for _, k, v in half:
    s = short(k)
    a = agg.setdefault(s, [0, 0.0])
    a[0] += 1; a[1] += v
tot = sum(v for _, _, v in half)
print(f"{'kernel':72s} {'n':>3s} {'us':>9s} {'share':>6s}")
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:72s} {c:3d} {v/1e3:9.1f} {100*v/tot:5.1f}%")
print(f"total {tot/1e3:.1f} us over {len(half)} launches")
