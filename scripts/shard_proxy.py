"""Scaling-floor proxy: step time of one traced GPU's shard of config 4 (what one rank of 8
processes) against the whole trace on one GPU, device-timed with CUDA events around K steps."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2512_08242_b200 as ch  # noqa: E402
import tracegen  # noqa: E402


def step_ms(b, p, K=20):
    st = torch.cuda.Stream()
    pipe = ch.Pipeline(b.cfg.n_gpus, len(b.labels), b.cfg.n_iters + 8, 1 << 15, device=0, stream=st)
    pipe.upload(b, b.n_counters, plan_laminar=True)
    for _ in range(3):
        pipe.run(p)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0, l0 = pipe.host_syncs(), pipe.launches()
    t = time.perf_counter()
    e0.record(st)
    for _ in range(K):
        pipe.run(p)
    e1.record(st)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t) / K * 1e3
    r = (e0.elapsed_time(e1) / K, wall, (pipe.host_syncs() - s0) / K, (pipe.launches() - l0) / K)
    pipe.close()
    return r


full = tracegen.generate(tracegen.config(4))
p = ch.default_params(full, full.labels, tracegen.workload_shapes(full.cfg), tracegen.op_kind)
for name, b in (("full trace", full), ("gpu 0 shard", full.gpu_slice([0]))):
    d, w, s, l = step_ms(b, p)
    print(f"{name:12s} events {b.n_events:9d} device {d:7.3f} ms  host wall {w:7.3f} ms  syncs {s:.0f} launches {l:.0f}")
