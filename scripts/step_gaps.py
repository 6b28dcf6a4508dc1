"""Where the bench step's wall time goes: device time of each ABI call (CUDA events on the ctx stream, gaps
included) vs host wall time of the Python call, for config 4 (one GPU).  Diagnostic only."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import tracegen
import paper_2512_08242_b200 as ch
from paper_2512_08242_b200 import pipeline as pl

b = tracegen.generate(tracegen.config(int(sys.argv[1]) if len(sys.argv) > 1 else 4))
p = ch.default_params(b, b.labels, tracegen.workload_shapes(b.cfg), tracegen.op_kind)
if len(sys.argv) > 2 and sys.argv[2] == "shard":      # traced GPU 0's shard (one rank of eight)
    b = b.gpu_slice([0])
stream = torch.cuda.Stream()
pipe = ch.Pipeline(b.cfg.n_gpus, len(b.labels), 256, 1 << 15, device=0, stream=stream)
pipe.upload(b, b.n_counters)
pipe.upload_cpu(*tracegen.cpu_samples(b.cfg.seed, int(b.t_l.min()), int(b.t_ke.max())))
ch.chopper_set_timing(pipe.ctx, True)
calls = ["load", "align", "attribute", "overlap", "breakdown", "reduce", "cpu"]
orig = {}
host = {k: 0.0 for k in calls}
dev = {k: 0.0 for k in calls}
evs = {}
def wrap(name, fn):
    def f(*a, **k):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t = time.perf_counter()
        r = fn(*a, **k)
        host[name] += time.perf_counter() - t
        e1.record(stream)
        evs.setdefault(name, []).append((e0, e1))
        return r
    return f
for name, attr in zip(calls, ["chopper_load_columns", "chopper_align", "chopper_attribute", "chopper_overlap",
                              "chopper_breakdown", "chopper_reduce_ranks", "chopper_cpu_util"]):
    setattr(pl, attr, wrap(name, getattr(pl, attr)))
for _ in range(3):
    pipe.run(p)
torch.cuda.synchronize()
for k in host: host[k] = 0.0
evs.clear()
K = 10
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record(stream)
w = time.perf_counter()
for _ in range(K):
    pipe.run(p)
t1.record(stream)
torch.cuda.synchronize()
w = (time.perf_counter() - w) / K * 1e3
tot = t0.elapsed_time(t1) / K
print(f"step device {tot:.3f} ms, wall {w:.3f} ms")
s = 0
for k in calls:
    d = sum(a.elapsed_time(b_) for a, b_ in evs.get(k, [])) / K
    s += d
    print(f"{k:10s} device {d:.3f} ms  host {host[k] / K * 1e3:.3f} ms")
print(f"sum of calls {s:.3f} ms; outside the calls {tot - s:.3f} ms")
