"""Key metrics of every launch in an ncu --set full report (the profiles/r02_ncu_*.txt summaries):
duration, DRAM bytes and throughput, L2 hit rate, achieved occupancy, registers, issue activity and the
top warp-stall reasons.  Usage: python scripts/ncu_summary.py REP [label]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, units = rows[0], rows[1]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
print(f"# ncu --set full summary of {rep}" + (f" ({sys.argv[2]})" if len(sys.argv) > 2 else ""))
for r in rows[2:]:
    d = dict(zip(h, r))
    u = dict(zip(h, units))
    print(f"\n## {d.get('Kernel Name', '?')[:110]}")
    for k in KEYS:
        if k in d:
            print(f"   {k:55s} {d[k]:>16s} {u.get(k, '')}")
    st = []
    for k in h:
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(d[k].replace(",", "")), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    st.sort(reverse=True)
    print("   top stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in st[:6]))
