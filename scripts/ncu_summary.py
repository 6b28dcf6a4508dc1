"""Summarize one `ncu --set full` capture (.ncu-rep) for profiles/: the roofline
numbers (duration, DRAM bytes, achieved GB/s), occupancy, issue activity and the
top warp-stall reasons.  Usage: python scripts/ncu_summary.py rep.ncu-rep [peak_gbs]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
peak = float(sys.argv[2]) if len(sys.argv) > 2 else 6548.2
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, unit, data = rows[0], rows[1], rows[2:]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__maximum_warps_per_active_cycle_pct", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1}
for v in data:
    name = v[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    print(f"kernel: {name}")
    vals = {}
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            x = float(v[i].replace(",", ""))
            vals[w] = x * SCALE.get(unit[i], 1)
            print(f"  {w:60s} {v[i]:>16s} {unit[i]}")
    if "gpu__time_duration.sum" in vals and "dram__bytes_read.sum" in vals:
        t = vals["gpu__time_duration.sum"]
        b = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
        print(f"  dram traffic {b / 1e6:.1f} MB in {t * 1e3:.3f} ms -> {b / t / 1e9:.1f} GB/s "
              f"({100 * b / t / 1e9 / peak:.1f}% of measured {peak} GB/s)")
    st = []
    for i, n in enumerate(hdr):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
            try:
                st.append((float(v[i].replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1
    print("  top stall reasons (pc samples): " +
          ", ".join(f"{n} {100 * x / tot:.0f}%" for x, n in sorted(st, reverse=True)[:6]))
