"""N>1 host logic on CPU (gloo, world_size 2): the sharding contract bench.py and the NCCL exchange rely on.

Rank r owns traced GPUs {g : g mod N == r}.  Per-GPU rows (instances ... GPU
rows, points, per-event outputs) depend only on that GPU's events, so every
rank computes them from its shard alone; only the clock offsets (a4) and the
global rows (a11) need the exchange.  Here each gloo rank runs the oracle on
its shard, the ranks all-gather their per-GPU rows (the role of NCCL
all-gather #2), and the gathered, re-indexed-by-gpu result must equal the
single-process run."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import oracle
    import tracegen
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = tracegen.config(3)
        cfg.n_iters, cfg.n_layers, cfg.n_gpus, cfg.opt_kernels, cfg.warmup = 2, 2, 4, 300, 0
        b = tracegen.generate(cfg)
        mine = [g for g in range(cfg.n_gpus) if g % world == rank]
        shard = b.gpu_slice(mine)
        p = oracle.default_params(b)
        o = oracle.run(shard, p)
        rows = {k: v for k, v in o.items() if k.split(".")[0] in ("inst", "layer", "phase", "iter", "point")}
        got = [None] * world
        dist.all_gather_object(got, (mine, rows))
        if rank == 0:
            whole = oracle.run(b, p)
            ok = True
            for t in ("inst", "layer", "phase", "iter", "point"):
                for f in ("busy", "prep", "call", "ovl", "n", "n_events", "phi"):
                    merged = {}
                    for (gs, r) in got:
                        for g in gs:
                            m = r[f"{t}.gpu"] == g
                            merged[g] = r[f"{t}.{f}"][m]
                    ref = whole[f"{t}.{f}"]
                    if t == "point":   # points are ordered (label, gpu, it): compare per gpu
                        for g in range(cfg.n_gpus):
                            if not np.array_equal(np.sort(merged[g]), np.sort(ref[whole["point.gpu"] == g])):
                                ok = False
                    else:
                        cat = np.concatenate([merged[g] for g in range(cfg.n_gpus)])
                        ok &= bool(np.array_equal(cat, ref))
            q.put(ok)
    finally:
        dist.destroy_process_group()


def test_two_rank_shards_reassemble():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True


def test_shard_ownership_covers_every_gpu():
    for world in (1, 2, 4, 8):
        owned = sorted(g for r in range(world) for g in range(8) if g % world == r)
        assert owned == list(range(8))
        per = [len([g for g in range(8) if g % world == r]) for r in range(world)]
        assert max(per) <= -(-8 // world)      # fits ceil(n_traced / nranks) exchange slots
