"""Summarise `ncu --set full` reports (scripts/round_ncu.sh) as the markdown
table in profiles/<round>/ncu_full_c3.md and the per-kernel DRAM traffic JSON
bench.py reads (profiles/ncu_traffic_c3.json).

    python scripts/ncu_summary.py gpurun_out/r1n4 profiles/round1/ncu_full_c3.md \
        profiles/ncu_traffic_c3.json
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
    src, md, js = sys.argv[1], sys.argv[2], sys.argv[3]
    lines = ["# ncu --set full --clock-control none, c3 training step (scripts/round_ncu.sh)", "",
             "Captured from `python scripts/profile_step.py --config c3 --steps 2` (eager step, "
             f"second step's launches); raw reports in {src} (not committed); table by "
             "`scripts/ncu_summary.py`.", "",
             "kernel | time us | DRAM read+write MB | " + " | ".join(c for c, _ in COLS[1:]) +
             " | grid x block", "---|" * (len(COLS) + 2) + "---"]
    traffic, gemm = {}, []
    for rep in ("full_fold", "full_fwd", "full_gemm"):
        for r in rows_of(f"{src}/{rep}.ncu-rep"):
            t = num(r["gpu__time_duration.sum"]) * TSCALE.get(r["gpu__time_duration.sum"][1], 1.0)
            dr = num(r["dram__bytes_read.sum"]) * SCALE.get(r["dram__bytes_read.sum"][1], 1)
            dw = num(r["dram__bytes_write.sum"]) * SCALE.get(r["dram__bytes_write.sum"][1], 1)
            k = short(r["Kernel Name"][0])
            vals = [f"{num(r[m]):.1f}" if m in r else "-" for _, m in COLS[1:]]
            lines.append(f"{k} | {t:.2f} | {(dr + dw) / 1e6:.1f} | " + " | ".join(vals) +
                         f" | {r['launch__grid_size'][0]} x {r['launch__block_size'][0]}")
            base = re.sub(r"<.*", "", k)
            if base == "tc_gemm_kernel":
                gemm.append(dr + dw)
            else:
                traffic[base] = dr + dw
    if gemm:
        traffic["tc_gemm_kernel"] = sum(gemm) / len(gemm)
    traffic["_source"] = ("ncu --set full --clock-control none (scripts/round_ncu.sh), c3 step, "
                          "DRAM read+write bytes per launch; tc_gemm_kernel = mean of the "
                          f"{len(gemm)} captured launches")
    open(md, "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(js, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
