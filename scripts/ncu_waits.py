"""mbarrier wait hot spots of a kernel from an `ncu --page source --csv
--print-source sass` dump: each try-wait loop (SYNCS...TRYWAIT + its retry
branch) with its share of the warp-stall samples and its barrier operand."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
f = lambda v: float(v) if v not in ("", None, "-") else 0.0
i = 0
while i < len(rows):
    if rows[i] and rows[i][0] == "Kernel Name":
        name, hdr = rows[i][1], rows[i + 1]
        j, data = i + 2, []
        while j < len(rows) and not (rows[j] and rows[j][0] == "Kernel Name"):
            if len(rows[j]) == len(hdr) and rows[j][0].startswith("0x"):
                data.append(rows[j])
            j += 1
        si = hdr.index("Warp Stall Sampling (All Samples)")
        tot = sum(f(r[si]) for r in data) or 1
        print("==", name[:90])
        for k, r in enumerate(data):
            if "SYNCS" in r[1] and "WAIT" in r[1]:
                s = sum(f(x[si]) for x in data[k:k + 4])
                print(f"  {s / tot * 100:5.1f}%  {r[0][-5:]}  {r[1].strip()[:70]}")
        print("  top:")
        for r in sorted(data, key=lambda r: -f(r[si]))[:10]:
            print(f"  {f(r[si]) / tot * 100:5.1f}%  {r[0][-5:]}  {r[1].strip()[:70]}")
        i = j
    else:
        i += 1
