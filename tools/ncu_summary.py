#!/usr/bin/env python
"""Summarise ncu --set full reports into profiles/ (markdown + traffic.json).

    python tools/ncu_summary.py --round r01 gpurun_out/prof_<workload>_<variant>.ncu-rep ...

Each report holds one launch of one kernel (captured with tools/prof_run.py).
The workload and variant are taken from the file name
(prof_<workload>_<variant>.ncu-rep).  traffic.json maps "<workload>:<variant>"
to dram__bytes_read.sum + dram__bytes_write.sum of that launch (bench.py's
roofline.traffic).
"""
import argparse
import csv
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__inst_executed_op_shfl.sum", "SHFL (warp inst)"),
    ("smsp__inst_executed_op_shared_ld.sum", "LDS (warp inst)"),
    ("smsp__inst_executed_op_global_ld.sum", "LDG (warp inst)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "Tbyte": 1e12}


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2]


def to_bytes(v, unit):
    try:
        return float(v) * SCALE.get(unit, 1.0)
    except ValueError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles"))
    ap.add_argument("reports", nargs="+")
    a = ap.parse_args()
    traffic_path = os.path.join(a.out, "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    lines = [f"# ncu --set full summaries ({a.round})", "",
             "One launch per report (tools/prof_run.py, after warm-up launches), "
             "`--clock-control none`, cold caches (ncu default cache control).", ""]
    for rep in a.reports:
        name = os.path.basename(rep).replace(".ncu-rep", "")
        m = re.match(r"prof_(.+)_(shuffle|plain)$", name)
        wl, var = (m.group(1), m.group(2)) if m else (name, "?")
        h, u, v = raw(rep)
        idx = {n: i for i, n in enumerate(h)}
        kern = v[idx["Kernel Name"]] if "Kernel Name" in idx else "?"
        lines += [f"## {wl} / {var}", "", f"kernel: `{kern[:160]}`", "", "| metric | value |",
                  "|---|---|"]
        for key, label in METRICS:
            if key in idx:
                lines.append(f"| {label} (`{key}`) | {v[idx[key]]} {u[idx[key]]} |")
        stalls = [(n.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v[i] or 0))
                  for n, i in idx.items()
                  if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")]
        tot = sum(s for _, s in stalls) or 1.0
        top = sorted(stalls, key=lambda x: -x[1])[:6]
        lines += ["", "stall samples: " + ", ".join(f"{n} {100 * s / tot:.1f}%" for n, s in top), ""]
        if "dram__bytes_read.sum" in idx and "dram__bytes_write.sum" in idx:
            rd = to_bytes(v[idx["dram__bytes_read.sum"]], u[idx["dram__bytes_read.sum"]])
            wr = to_bytes(v[idx["dram__bytes_write.sum"]], u[idx["dram__bytes_write.sum"]])
            if rd is not None and wr is not None:
                traffic[f"{wl}:{var}"] = rd + wr
    os.makedirs(a.out, exist_ok=True)
    out = os.path.join(a.out, f"{a.round}_ncu_summary.md")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    print(out, traffic_path)


if __name__ == "__main__":
    main()
