"""Summarise `ncu --set full` reports (scripts/round2_ncu.sh) as a markdown
table for profiles/<round>/ and the per-kernel DRAM traffic JSON bench.py
reads for the `roofline.traffic` field (profiles/ncu_traffic_<config>.json).

    python scripts/ncu_summary.py c3 profiles/round2/ncu_full_c3.md \
        profiles/ncu_traffic_c3.json gpurun_out/r2n/c3_fold.ncu-rep ...
"""
import csv, io, json, re, subprocess, sys

COLS = [("time", "gpu__time_duration.sum"),
        ("DRAM %", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        ("L2 %", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("L1/smem %", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("SM %", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("tensor pipe % (active)", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
        ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("regs", "launch__registers_per_thread")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TSCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        yield {k: (v, u) for k, v, u in zip(h, r, units)}


def num(cell):
    return float(cell[0].replace(",", "")) if cell and cell[0] not in ("", "n/a") else float("nan")


def short(name):
    name = re.sub(r"\(.*", "", name).replace("void ", "")
    return re.sub(r"\(anonymous namespace\)::|unnamed>::", "", name).strip()


def main():
    cfg, md, js, reps = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4:]
    lines = [f"# ncu --set full --clock-control none, {cfg} training step (scripts/round2_ncu.sh)",
             "",
             f"Captured from `python scripts/profile_step.py --config {cfg} --steps 2` (eager "
             "step, second step's launches) after a clean plain run of the same command; "
             "table by `scripts/ncu_summary.py`.  Cold-cache, serialised: compare shares and "
             "traffic, not absolute step time.", "",
             "kernel | time us | DRAM read+write MB | " + " | ".join(c for c, _ in COLS[1:]) +
             " | grid x block", "---|" * (len(COLS) + 2) + "---"]
    per = {}
    for rep in reps:
        for r in rows_of(rep):
            t = num(r["gpu__time_duration.sum"]) * TSCALE.get(r["gpu__time_duration.sum"][1], 1.0)
            dr = num(r["dram__bytes_read.sum"]) * SCALE.get(r["dram__bytes_read.sum"][1], 1)
            dw = num(r["dram__bytes_write.sum"]) * SCALE.get(r["dram__bytes_write.sum"][1], 1)
            k = short(r["Kernel Name"][0])
            vals = [f"{num(r[m]):.1f}" if m in r else "-" for _, m in COLS[1:]]
            lines.append(f"{k} | {t:.2f} | {(dr + dw) / 1e6:.1f} | " + " | ".join(vals) +
                         f" | {r['launch__grid_size'][0]} x {r['launch__block_size'][0]}")
            per.setdefault(re.sub(r"<.*", "", k), []).append(dr + dw)
    traffic = {k: sum(v) / len(v) for k, v in per.items()}
    traffic["_source"] = (f"ncu --set full --clock-control none (scripts/round2_ncu.sh), {cfg} "
                          "step, DRAM read+write bytes per launch (mean over the captured "
                          "launches of each kernel)")
    open(md, "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(js, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
