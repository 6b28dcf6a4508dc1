"""summarize an iteration directory: tests, bench phases, ncu key metrics"""
import csv, json, sys
d = sys.argv[1]
print(open(f"{d}/tests.log").read().strip().splitlines()[-2:])
try:
    b = json.loads(open(f"{d}/bench.log").read().strip().splitlines()[-1])
    r = b["roofline"]
    print("ms/step", round(b["ms_per_step"], 3), "ev kernel", round(r["avg_launch_ms"], 4), "frac", round(r["frac"], 3),
          {k: round(v, 3) for k, v in r["phase_ms_last_step"].items() if v})
except Exception as e:
    print("bench:", e, open(f"{d}/bench.log").read()[-800:])
try:
    rows = list(csv.reader(open(f"{d}/prof_details.csv")))
    h = rows[0]
    i_n, i_v, i_u = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    want = ["Duration", "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
            "Achieved Occupancy", "Executed Instructions", "L1/TEX Hit Rate", "Warp Cycles Per Issued Instruction",
            "Eligible Warps Per Scheduler", "Dynamic Shared Memory Per Block"]
    for x in rows[1:]:
        if x[i_n] in want:
            print("  ", x[i_n], x[i_v], x[i_u])
except Exception as e:
    print("ncu:", e)
