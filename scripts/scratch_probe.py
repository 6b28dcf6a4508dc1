"""Scratch high-water and step time per config (one GPU): python scripts/scratch_probe.py [cids...]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2512_08242_b200 as ch  # noqa: E402
import tracegen  # noqa: E402
from tracegen import stress  # noqa: E402

for arg in sys.argv[1:] or ["1", "2", "3", "4", "5s"]:
    t = time.time()
    if arg == "5s":
        cfg = tracegen.config(5)
        b = stress.generate(cfg, gpus=[0], threads=16)
    else:
        cfg = tracegen.config(int(arg))
        b = tracegen.generate(cfg)
    tg = time.time() - t
    p = oracle.default_params(b)
    pipe = ch.Pipeline(cfg.n_gpus, len(b.labels), max(cfg.n_iters + 3, 8), 1 << 15, device=0)
    pipe.upload(b, b.n_counters)
    for full in (False, True):
        res = pipe.run(p, full=full)
        torch.cuda.synchronize()
        t0 = time.time()
        for _ in range(3):
            res = pipe.run(p, full=full)
        torch.cuda.synchronize()
        dt = (time.time() - t0) / 3
        lv = (b.span_gl & 0xFF)
        print(f"config {arg} full={full}: N={b.n_events} S={len(b.span_gl)} S_lv={np.bincount(lv, minlength=4).tolist()} "
              f"C={b.n_counters} inst={int(res['tables'].inst.n)} layer={int(res['tables'].layer.n)} "
              f"high={ch.load_library().chopper_scratch_used(pipe.ctx) / 1e9:.3f} GB "
              f"({ch.load_library().chopper_scratch_used(pipe.ctx) / max(b.n_events, 1):.1f} B/event) "
              f"scratch_bytes={pipe.scratch.numel() / 1e9:.2f} GB step={dt * 1e3:.2f} ms gen={tg:.1f}s", flush=True)
    pipe.close()
    del pipe, b
    torch.cuda.empty_cache()
