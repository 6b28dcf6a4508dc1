"""Summarize an ncu launch list (gpu__time_duration.sum) of bench.py: per-kernel time of the last step."""
import collections
import csv
import re
import sys

path = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4     # warm-up steps + timed steps in the capture
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h, data = rows[hi], rows[hi + 1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
last = data[-(len(data) // steps):]
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in last:
    v = float(r[vi].replace(",", ""))
    v = v * 1e3 if r[ui] == "usecond" else v * 1e6 if r[ui] == "msecond" else v
    m = re.search(r"(k_[a-z0-9_]+)", r[ki])
    k = m.group(1) if m else r[ki][:50]
    tot[k] += v
    cnt[k] += 1
s = sum(tot.values())
print(f"launches in last step: {len(last)}, kernel time {s / 1e6:.3f} ms")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    print(f"{v / 1e6:8.3f} ms {100 * v / s:5.1f}% x{cnt[k]:4d} {k}")
