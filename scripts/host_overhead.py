"""Host-side cost of one step on a small shard: wall time per ABI call (each call is followed by a stream
synchronize), the Python marshalling share, and the device phase times."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2512_08242_b200 as ch  # noqa: E402
from paper_2512_08242_b200 import pipeline as pl  # noqa: E402
import tracegen  # noqa: E402

full = tracegen.generate(tracegen.config(4))
p = ch.default_params(full, full.labels, tracegen.workload_shapes(full.cfg), tracegen.op_kind)
b = full.gpu_slice([0])
st = torch.cuda.Stream()
pipe = ch.Pipeline(8, len(b.labels), 208, 1 << 15, device=0, stream=st)
pipe.upload(b, b.n_counters, plan_laminar=True)
ch.chopper_set_timing(pipe.ctx, True)
for _ in range(5):
    pipe.run(p)
torch.cuda.synchronize()
# time the whole run() and python-side pieces
K = 30
t = time.perf_counter()
for _ in range(K):
    pipe.run(p)
torch.cuda.synchronize()
print(f"run() wall {1e3 * (time.perf_counter() - t) / K:.3f} ms")
print({n: round(ch.chopper_phase_time(pipe.ctx, i) or 0, 3) for i, n in enumerate(ch.PHASES)})
import cProfile, pstats
cProfile.run("for _ in range(10): pipe.run(p)", "/tmp/hp")
pstats.Stats("/tmp/hp").sort_stats("tottime").print_stats(15)
