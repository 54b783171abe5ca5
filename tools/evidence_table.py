#!/usr/bin/env python
"""Per-stencil evidence table from the committed ncu summaries.

    python tools/evidence_table.py [--round r01]  -> markdown on stdout

Reads profiles/<round>_ncu_summary.md (one ncu --set full launch per
workload x variant) and profiles/<round>_ops/ops_<w>_<v>.txt (dynamic SASS
opcode counts, tools/ncu_ops.py).  DRAM / compulsory = (dram read + write)
/ (interior points x compulsory bytes per point) of that launch; *_pair rows
are two-sweep k2d2 launches (instr / pt per point of the launch = per two
sweeps).
"""
import argparse
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# interior points of one launch and compulsory bytes per point
PTS = {"gaussblur": 8188 ** 2, "jacobi2d_paper": 32766 ** 2, "gameoflife": 16382 ** 2,
       "laplacian": 510 ** 3, "wave13pt": 508 ** 3, "jacobi3d": 1022 ** 3, "divergence": 510 ** 3,
       "gradient": 510 ** 3, "tricubic": 253 ** 3,
       # two-sweep (k2d2) launches: one read and one write per launch, 2 sweeps
       "jacobi2d_pair": 32766 ** 2, "gameoflife_pair": 16382 ** 2,
       "jacobi2d_paper_pair": 32766 ** 2, "gaussblur_pair": 8188 ** 2}
BPP = {"gaussblur": 8, "jacobi2d_paper": 8, "gameoflife": 8, "laplacian": 16, "wave13pt": 24,
       "jacobi3d": 8, "divergence": 16, "gradient": 16, "tricubic": 20, "jacobi2d_pair": 8,
       "gameoflife_pair": 8, "jacobi2d_paper_pair": 8, "gaussblur_pair": 8}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TSCALE = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}


def val(sec, label):
    m = re.search(r"\| " + re.escape(label) + r" \(`[^`]+`\) \| ([\d.]+) (\S+)", sec)
    return (float(m.group(1)), m.group(2)) if m else (None, None)


def ops(rnd, wl, var):
    p = os.path.join(ROOT, "profiles", f"{rnd}_ops", f"ops_{wl}_{var}.txt")
    out = {}
    if os.path.exists(p):
        for line in open(p):
            t = line.split()
            if len(t) >= 2 and t[1].isdigit():
                out[t[0]] = int(t[1])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    a = ap.parse_args()
    s = open(os.path.join(ROOT, "profiles", f"{a.round}_ncu_summary.md")).read()
    print("| workload / variant | ncu time (ms) | DRAM / compulsory | DRAM GB/s | L2 hit % | regs | warps active % "
          "| issue active % | instr / pt | SHFL / pt | LDS / pt | top-3 stalls |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for sec in s.split("## ")[1:]:
        name = sec.split("\n")[0].strip()
        wl, var = name.split(" / ")
        if wl not in PTS:
            continue
        d, du = val(sec, "duration")
        rd, ru = val(sec, "dram read")
        wr, wu = val(sec, "dram write")
        l2, _ = val(sec, "L2 hit %")
        regs, _ = val(sec, "regs/thread")
        occ, _ = val(sec, "warps active %")
        iss, _ = val(sec, "issue active %")
        inst, _ = val(sec, "warp instructions")
        ms = d * TSCALE[du]
        dram = rd * SCALE[ru] + wr * SCALE[wu]
        comp = PTS[wl] * BPP[wl]
        o = ops(a.round, wl, var)
        n = PTS[wl] / 32.0
        m = re.search(r"stall samples: (.*)", sec)
        st = ", ".join(x.rsplit(" ", 1)[0] for x in m.group(1).split(", ")[:3]) if m else ""
        print(f"| {wl} / {var} | {ms:.3f} | {dram / comp:.2f} | {dram / (ms * 1e-3) / 1e9:.0f} | {l2:.1f} | {regs:.0f} "
              f"| {occ:.0f} | {iss:.0f} | {inst / n:.1f} | {o.get('SHFL', 0) / n:.2f} | {o.get('LDS', 0) / n:.2f} | {st} |")


if __name__ == "__main__":
    main()
