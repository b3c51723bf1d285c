"""Top SASS lines by warp-stall samples from an `ncu --page source --csv
--print-source sass` dump (one or more kernels)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
i = 0
while i < len(rows):
    if rows[i] and rows[i][0] == "Kernel Name":
        name = rows[i][1]
        hdr = rows[i + 1]
        j = i + 2
        data = []
        while j < len(rows) and not (rows[j] and rows[j][0] == "Kernel Name"):
            if len(rows[j]) == len(hdr):
                data.append(rows[j])
            j += 1
        si = hdr.index("Warp Stall Sampling (All Samples)")
        f = lambda v: float(v) if v not in ("", None) else 0.0
        tot = sum(f(r[si]) for r in data) or 1
        stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        print("==", name[:100], "samples", tot)
        agg = {h: sum(f(r[hdr.index(h)]) for r in data) for h in stalls}
        print("   by reason:", [(k, round(v / tot * 100, 1)) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:6]])
        for r in sorted(data, key=lambda r: -f(r[si]))[:n]:
            st = sorted(((h, f(r[hdr.index(h)])) for h in stalls), key=lambda x: -x[1])[:2]
            print("  ", r[0], f"{f(r[si]) / tot * 100:5.1f}%", r[1][:70], [(a[6:], int(b)) for a, b in st])
        i = j
    else:
        i += 1
