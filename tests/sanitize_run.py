"""Workload for the compute-sanitizer test (tests/test_gpu_sanitizer.py): config 1 plus two small seeded
traces -- one FSDP-shaped (the lean a2 path), one with three compute streams per GPU and crossing spans (the
general partition / sort path and the exact sweep) -- through all six calls in full mode, each checked
against the oracle so a silent corruption also fails."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import tracegen  # noqa: E402
from parity import assert_parity, run_both  # noqa: E402
from tinytrace import TinyTrace, params  # noqa: E402


def multi_stream_trace(seed):
    rng = np.random.default_rng(seed)
    tt = TinyTrace(n_gpus=2, labels=["a", "b", "c"])
    evs = []
    for g in range(2):
        tt.span(g, 0, 0, 10 ** 6, 5).span(g, 1, 100, 400_000, 0).span(g, 1, 300_000, 900_000, 1)  # crossing phases
        for q in range(30):
            s0 = int(rng.integers(0, 900_000))
            tt.span(g, 3, s0, s0 + int(rng.integers(100, 50_000)), int(rng.integers(0, 3)))
        for st in range(3):
            t = 1000 + 37 * st
            for _ in range(200):
                d = int(rng.integers(5, 2000))
                evs.append((g, t - int(rng.integers(0, 400)), t, t + d, st, 0))
                t += d + int(rng.integers(0, 500))
        t = 500
        for k in range(40):
            d = int(rng.integers(100, 5000))
            evs.append((g, t - 100, t, t + d, 4 + (k % 2), 1 + (k % 2)))
            t += d + int(rng.integers(0, 20_000))
    for (g, tl, ks, ke, st, kind) in sorted(evs, key=lambda e: (e[0], e[1])):
        tt.ev(g, tl, ks, ke, kind=kind, stream=st)
    for g in range(2):
        tt.sample(g, 0, 1500, 300_000).sample(g, 400_000, 1800, 350_000)
    return tt.bundle()


def main():
    b1 = tracegen.generate(tracegen.config(1))
    cfg = tracegen.config(3)
    cfg.n_iters, cfg.n_layers, cfg.n_gpus, cfg.opt_kernels, cfg.warmup = 2, 2, 2, 200, 0
    b2 = tracegen.generate(cfg)
    b3 = multi_stream_trace(5)
    for b, p in ((b1, None), (b2, None), (b3, params(b3, op_type=np.array([1, 2, 0], np.int32)))):
        ref, got, res, pipe = run_both(b, p)
        assert_parity(ref, got)
        pipe.close()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
