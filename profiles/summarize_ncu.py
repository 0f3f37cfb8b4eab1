"""Summarises an ncu --set full report (.ncu-rep) into profiles/: per-kernel
duration, DRAM bytes, achieved DRAM bandwidth, occupancy and registers.

    python profiles/summarize_ncu.py gpurun_out/prof_c2.ncu-rep profiles/r01_c2_ncu_full
"""
import csv
import json
import subprocess
import sys

FIELDS = {
    "time_us": "gpu__time_duration.sum",
    "dram_read_mb": "dram__bytes_read.sum",
    "dram_write_mb": "dram__bytes_write.sum",
    "dram_pct_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct_peak": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_per_sm": "sm__warps_active.avg.per_cycle_active",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
}


def main(rep, out_prefix):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        rec = {"kernel": r[hdr.index("Kernel Name")]}
        for k, m in FIELDS.items():
            if m in hdr:
                v = r[hdr.index(m)].replace(",", "")
                u = units[hdr.index(m)]
                try:
                    x = float(v)
                except ValueError:
                    rec[k] = v
                    continue
                if k == "time_us":
                    x = x / 1000.0 if u == "ns" else (x * 1000.0 if u == "ms" else x)
                if k.endswith("_mb"):
                    x = x / 1e6 if u == "byte" else (x * 1000.0 if u == "Gbyte" else (x / 1000.0 if u == "Kbyte" else x))
                rec[k] = x
        t = rec.get("time_us") or 0
        rec["dram_gbs"] = (rec.get("dram_read_mb", 0) + rec.get("dram_write_mb", 0)) * 1e6 / (t * 1e-6) / 1e9 if t else None
        out.append(rec)
    json.dump(out, open(out_prefix + ".json", "w"), indent=1)
    with open(out_prefix + ".md", "w") as f:
        f.write(f"ncu --set full summary of `{rep}` (cold-cache, serialised replays: compare shares, not absolutes)\n\n")
        f.write("| kernel | us | DRAM rd MB | DRAM wr MB | DRAM GB/s | DRAM % | SM % | warps/SM | regs | grid |\n|---|---|---|---|---|---|---|---|---|---|\n")
        for rec in out:
            f.write("| {} | {:.1f} | {:.1f} | {:.1f} | {:.0f} | {:.1f} | {:.1f} | {:.1f} | {} | {} |\n".format(
                rec["kernel"][:60], rec.get("time_us", 0), rec.get("dram_read_mb", 0), rec.get("dram_write_mb", 0),
                rec.get("dram_gbs") or 0, rec.get("dram_pct_peak", 0), rec.get("sm_pct_peak", 0),
                rec.get("warps_active_per_sm", 0), rec.get("registers", ""), rec.get("grid", "")))
    print(open(out_prefix + ".md").read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
