"""Per-CUDA-line totals from an ncu report (ncu -i REP --page source --print-source cuda,sass --csv):
warp instructions executed, stall samples, local-memory sectors.  usage: src_lines.py REP [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f = None; hdr = None; agg = {}; tot_i = 0; tot_s = 0
for r in csv.reader(io.StringIO(txt)):
    if not r: continue
    if r[0] == "File Path": f = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if r[0] == "Function Name" or hdr is None: continue
    if r[0] != "":            # a source line row (aggregated)
        d = dict(zip(hdr[2:], r[2:]))
        try:
            ins = int(float(d.get("Instructions Executed", "0") or 0)); smp = int(float(d.get("Warp Stall Sampling (All Samples)", "0") or 0))
            loc = int(float(d.get("L2 Theoretical Sectors Local", "0") or 0))
        except ValueError:
            continue
        key = (f, int(r[0])); a = agg.setdefault(key, [0, 0, 0, r[1].strip()[:90]])
        a[0] += ins; a[1] += smp; a[2] += loc; tot_i += ins; tot_s += smp
print(f"total warp inst {tot_i:,}  samples {tot_s:,}")
for (fn, ln), (i, s, l, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{fn}:{ln:5d} inst {i:11,d} ({100*i/max(tot_i,1):4.1f}%) smp {100*s/max(tot_s,1):4.1f}% loc {l:8d} | {src}")
