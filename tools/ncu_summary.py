"""Summarise ncu captures into profiles/<round>/ (development tool, run here, no GPU).

    python tools/ncu_summary.py r1 gpurun_out/prof_guarded.ncu-rep [more.ncu-rep ...] \
        [--launches gpurun_out/launches.csv]

Writes profiles/<round>/SUMMARY.md (per-kernel duration, DRAM bytes, throughput,
registers, occupancy) and merges per-launch DRAM traffic into profiles/traffic.json,
which bench.py reports as roofline.traffic.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
}
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "us": 1e-6, "ms": 1e-3, "ns": 1e-9,
         "Ghz": 1e9, "Mhz": 1e6}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0].replace("void ", "").split("::")[-1]}
        for i, name in enumerate(h):
            if name in WANT:
                v = r[i].replace(",", "")
                try:
                    v = float(v) * SCALE.get(units[i], 1.0)
                except ValueError:
                    pass
                d[WANT[name]] = v
        res.append(d)
    return res


def main():
    rnd, args = sys.argv[1], sys.argv[2:]
    launches = None
    if "--launches" in args:
        i = args.index("--launches")
        launches = args[i + 1]
        args = args[:i] + args[i + 2:]
    outdir = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(outdir, exist_ok=True)
    lines = [f"# ncu summary ({rnd})", "", "From `ncu --set full --clock-control none` captures "
             "(cold L2, serialised; compare shares, not absolutes, with bench.py).", "",
             "| kernel | capture | us | DRAM read MB | DRAM write MB | GB/s (DRAM) | DRAM % peak | regs | grid x block | warps active % |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for rep in args:
        for d in raw_rows(rep):
            dur = d.get("duration", float("nan"))
            rd, wr = d.get("dram_read", 0.0), d.get("dram_write", 0.0)
            lines.append(f"| {d['kernel']} | {os.path.basename(rep)} | {dur * 1e6:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | "
                         f"{(rd + wr) / dur / 1e9:.0f} | {d.get('dram_pct_peak', float('nan')):.1f} | {d.get('regs', '')} | "
                         f"{int(d.get('grid', 0))} x {int(d.get('block', 0))} | {d.get('warps_active_pct', float('nan')):.1f} |")
            traffic[d["kernel"]] = rd + wr
    if launches:
        rows = list(csv.reader(open(launches)))
        hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
        h = rows[hi]
        ki, vi = h.index("Kernel Name"), h.index("Metric Value")
        per = defaultdict(list)
        for r in rows[hi + 1:]:
            if "lmsgd" in r[ki]:
                per[r[ki].split("(")[0].replace("void ", "").split("::")[-1]].append(float(r[vi].replace(",", "")))
        tot = sum(sum(v) for v in per.values())
        lines += ["", f"Launch list ({os.path.basename(launches)}, `--metrics gpu__time_duration.sum`):", "",
                  "| kernel | launches | mean us | share of lmsgd time |", "|---|---|---|---|"]
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot:.3f} |")
    open(os.path.join(outdir, "SUMMARY.md"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
