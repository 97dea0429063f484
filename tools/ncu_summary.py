"""Summarise an `ncu --set full` report and an ncu launch list into profiles/.

  python tools/ncu_summary.py --rep gpurun_out/r01_prof.ncu-rep --launches gpurun_out/r01_launches.csv \
      --tag r01 --config 3

Writes profiles/<tag>_ncu_summary.md (human-readable) and profiles/ncu_k4_summary.json (the K4 DRAM
traffic per launch that bench.py reports as roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe active %"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", "DMMA instructions"),
    ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "shared pipe (fp64+tensor) %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("smsp__inst_executed.sum", "instructions"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def to_bytes(v, u):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--config", type=int, default=3)
    a = ap.parse_args()
    hdr, units, rows = raw(a.rep)
    col = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu summary {a.tag} (config {a.config}; `ncu --set full --clock-control none`, "
             f"tools/run_step.py)\n", "| kernel | " + " | ".join(n for _, n in METRICS) + " |",
             "|---|" + "---|" * len(METRICS)]
    k4 = []
    for r in rows:
        name = r[col["Kernel Name"]].split("(")[0]
        vals = []
        for m, _ in METRICS:
            if m in col:
                vals.append(f"{r[col[m]]} {units[col[m]]}".strip())
            else:
                vals.append("n/a")
        lines.append(f"| {name} | " + " | ".join(vals) + " |")
        if "k4_contract" in name:
            k4.append(to_bytes(r[col["dram__bytes_read.sum"]], units[col["dram__bytes_read.sum"]]) +
                      to_bytes(r[col["dram__bytes_write.sum"]], units[col["dram__bytes_write.sum"]]))
    if a.launches:
        lines += ["", "## launch list (ncu gpu__time_duration.sum, cold-cache serialised: compare shares)", "",
                  "| kernel | launches | mean µs | share |", "|---|---|---|---|"]
        tot = defaultdict(list)
        rows2 = list(csv.reader(open(a.launches)))
        h2 = None
        for r in rows2:
            if r and r[0] == "ID":
                h2 = {k: i for i, k in enumerate(r)}
                continue
            if h2 and len(r) == len(h2):
                v = float(r[h2["Metric Value"]].replace(",", ""))
                unit = r[h2["Metric Unit"]]
                us = v / 1e3 if unit in ("nsecond", "ns") else (v if unit in ("usecond", "us") else v * 1e3)
                tot[r[h2["Kernel Name"]].split("(")[0]].append(us)
        s = sum(sum(v) for v in tot.values())
        for k, v in sorted(tot.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {sum(v) / s:.3f} |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"{a.tag}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
    if k4:
        p = os.path.join(ROOT, "profiles", "ncu_k4_summary.json")
        d = json.load(open(p)) if os.path.exists(p) else {}
        d[f"config{a.config}"] = {"dram_bytes_per_launch": int(sum(k4) / len(k4)), "source": a.rep, "tag": a.tag}
        json.dump(d, open(p, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
