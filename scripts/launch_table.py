"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) as a
markdown table: per-kernel launch count, device time and share of the
library's step time.  torch's own launches (the L2-flush fills between timed
steps, outside the timed events, and the table initialisation) are excluded.

    python scripts/launch_table.py launches.csv [title] > table.md
"""
import collections, csv, re, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
recs = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hdr_i + 1:]
        if len(r) > vi and r[mi] == "gpu__time_duration.sum"]


def short(k):
    k = re.sub(r"\(.*", "", k).replace("void ", "")
    return k.replace("dlrm::<unnamed>::", "").replace("dlrm::(anonymous namespace)::", "")[:64]


agg = collections.OrderedDict()
flush = 0.0
for k, v in recs:
    if k.startswith("void at::") or k.startswith("at::"):  # torch: L2 flush fills, table init
        flush += v
        continue
    a = agg.setdefault(short(k), [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
title = sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]
print(f"# {title}\n")
print("Per-launch device times are cold-cache and serialised under ncu: compare SHARES, "
      "not absolute times.\n")
print("kernel | launches | total us | share")
print("---|---|---|---")
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k} | {c} | {v / 1e3:.1f} | {100 * v / tot:.1f}%")
print(f"\ntotal {tot / 1e3:.1f} us over {sum(a[0] for a in agg.values())} launches "
      f"(+ {flush / 1e3:.1f} us of torch L2-flush / init kernels, excluded)")
