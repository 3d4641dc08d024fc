#!/usr/bin/env python
"""Summarise Nsight Compute output into a small markdown file for profiles/.

    python tools/profile_summary.py --rep gpurun_out/prof.ncu-rep \
        [--launches gpurun_out/launches.csv] --title "r1 ..." > profiles/r1_x.md

--rep       an `ncu --set full` capture: per-kernel duration, DRAM bytes, pipe
            utilisation, issue activity, occupancy, top stall reasons and the
            hottest SASS lines (needs --import-source / -lineinfo).
--launches  a `--metrics gpu__time_duration.sum` launch list: per-kernel count,
            total / mean device time and share of the listed time.
"""
import argparse
import collections
import csv
import io
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg", "SM cycles elapsed"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "FMA-heavy pipe busy % (elapsed)"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe busy %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes_read.sum.per_second", "DRAM read bandwidth"),
    ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps / scheduler"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def run(cmd):
    return subprocess.run(cmd, capture_output=True, text=True).stdout


def rep_summary(rep):
    out = run(["ncu", "-i", rep, "--page", "raw", "--csv"])
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        lines.append(f"### {d.get('Kernel Name', '?')}\n")
        lines.append("| metric | value | unit |\n|---|---|---|")
        for k, name in KEYS:
            if k in d:
                lines.append(f"| {name} (`{k}`) | {d[k]} | {u.get(k, '')} |")
        st = []
        for k in hdr:
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(d[k]), k))
                except ValueError:
                    pass
        lines.append("\nTop stall reasons (warps per issued instruction):\n")
        for v, k in sorted(st, reverse=True)[:8]:
            name = k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")
            lines.append(f"- {name}: {v:.3f}")
        lines.append("")
    src = run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"])
    srows = list(csv.reader(io.StringIO(src)))
    if len(srows) > 2:
        h = srows[1]
        try:
            iS = h.index("Warp Stall Sampling (All Samples)")
            iSrc = h.index("Source")
            body = srows[2:]
            tot = sum(int(r[iS]) for r in body if len(r) > iS and r[iS].isdigit())
            lines.append(f"Hottest SASS lines ({tot} stall samples):\n")
            lines.append("| samples | % | instruction |\n|---|---|---|")
            top = sorted((r for r in body if len(r) > iS and r[iS].isdigit()),
                         key=lambda r: -int(r[iS]))[:12]
            for r in top:
                lines.append(f"| {r[iS]} | {100 * int(r[iS]) / max(tot, 1):.1f} | `{r[iSrc].strip()}` |")
        except ValueError:
            pass
    return "\n".join(lines)


def launches_summary(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    iK, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= iV:
            continue
        name = r[iK].split("(")[0]
        v = float(r[iV].replace(",", ""))
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    total = sum(t for _, t in agg.values())
    lines = ["| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {n} | {t / 1e3:.1f} | {t / n / 1e3:.2f} | {100 * t / total:.1f}% |")
    return "\n".join(lines)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--title", default="profile")
    ap.add_argument("--cmd", default="")
    a = ap.parse_args()
    print(f"# {a.title}\n")
    if a.cmd:
        print(f"Command: `{a.cmd}`\n")
    if a.launches:
        print("## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`; "
              "cold-cache, serialised: compare shares)\n")
        print(launches_summary(a.launches))
        print()
    if a.rep:
        print("## `ncu --set full` capture\n")
        print(rep_summary(a.rep))


if __name__ == "__main__":
    main()
