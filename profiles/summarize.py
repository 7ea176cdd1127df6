"""Summarise ncu output into profiles/<tag>_*.md.

    python profiles/summarize.py launches <launches.csv> <tag>
    python profiles/summarize.py full <report.ncu-rep> <tag>
"""
import collections
import csv
import io
import re
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent


def launches(path, tag):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        v = float(d["Metric Value"]) * {"usecond": 1e3, "msecond": 1e6}.get(d["Metric Unit"], 1)
        k = re.sub(r"\(.*", "", d["Kernel Name"]).replace("tfem::<unnamed>::", "")
        agg.setdefault(k, []).append(v)
    tot = sum(sum(v) for v in agg.values())
    out = [f"# {tag}: kernel launch list (ncu gpu__time_duration, cold cache, serialised)",
           "", f"source: `{Path(path).name}`; shares are of all profiled launches.  CG "
           "launches after the solve's last iteration exit at once (graph overshoot), so "
           "the median is the per-launch cost.", "",
           "| kernel | launches | median us | avg us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        med = sorted(v)[len(v) // 2]
        out.append(f"| `{k}` | {len(v)} | {med / 1e3:.1f} | {sum(v) / len(v) / 1e3:.1f} | "
                   f"{100 * sum(v) / tot:.1f}% |")
    (HERE / f"{tag}_launches.md").write_text("\n".join(out) + "\n")
    print("\n".join(out))


METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "blocks/SM (reg limit)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
     "long-scoreboard stall/issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "wait stall/issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
     "short-scoreboard stall/issue"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps/scheduler"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def full(path, tag):
    """path: an .ncu-rep, or the `--page raw --csv` export of one."""
    if str(path).endswith(".csv"):
        raw = Path(path).read_text()
    else:
        raw = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"],
                             capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = [f"# {tag}: ncu --set full summary", "", f"source: `{Path(path).name}`", ""]
    for r in rows[2:]:
        name = re.sub(r"\(.*", "", r[hdr.index("Kernel Name")]).replace("unnamed>::", "")
        out.append(f"## `{name}`")
        out.append("")
        out.append("| metric | value |")
        out.append("|---|---|")
        for m, label in METRICS:
            if m in hdr:
                i = hdr.index(m)
                out.append(f"| {label} (`{m}`) | {r[i]} {units[i]} |")
        out.append("")
    (HERE / f"{tag}_ncu_full.md").write_text("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
