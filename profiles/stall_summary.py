"""Per-kernel warp-stall breakdown from an ncu --set full report: the PC-sampling
stall counters (smsp__pcsamp_warps_issue_stalled_*) as shares of all samples,
plus issue-slot use, for each profiled launch whose name matches a filter.

    python profiles/stall_summary.py rep.ncu-rep [regex] > out.md
"""
import csv
import re
import subprocess
import sys


def main(rep, pat=".*"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr = rows[0]
    stall = [i for i, h in enumerate(hdr)
             if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
    extra = ["gpu__time_duration.sum", "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
             "sm__warps_active.avg.per_cycle_active", "launch__grid_size", "launch__registers_per_thread"]
    rx = re.compile(pat)
    print("| launch | kernel | " + " | ".join(e.split("__")[1] for e in extra) + " | top stalls (share of samples) |")
    print("|---|---|" + "---|" * len(extra) + "---|")
    for n, r in enumerate(rows[2:]):
        name = r[hdr.index("Kernel Name")]
        if not rx.search(name):
            continue
        vals = []
        for i in stall:
            try:
                vals.append((float(r[i].replace(",", "")), hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
        tot = sum(v for v, _ in vals) or 1.0
        top = sorted(vals, reverse=True)[:7]
        ex = []
        for e in extra:
            ex.append(r[hdr.index(e)] if e in hdr else "")
        print(f"| {n} | {name[:40]} | " + " | ".join(ex) + " | " +
              ", ".join(f"{k} {100 * v / tot:.0f}%" for v, k in top) + " |")


if __name__ == "__main__":
    main(*sys.argv[1:])
