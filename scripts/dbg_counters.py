import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_gpu_parity as T
from parity import run_both
from tinytrace import TinyTrace, params, AG, RS
rng = np.random.default_rng(77)
G = 2
tt = TinyTrace(n_gpus=G, n_counters=2, labels=["l%d" % i for i in range(4)])
for g in range(G):
    n = 4500 + 700 * g
    t = 1000
    tt.span(g, 0, 0, 10 ** 9, 7); tt.span(g, 1, 0, 10 ** 9, 0)
    names = []
    for k in range(n):
        d = int(rng.integers(50, 400)); tl = t - int(rng.integers(0, 30)); ks = t
        tt.ev(g, tl, ks, ks + d, name=k % 3); names.append(k % 3)
        tt.span(g, 3, tl - 1, tl + 1, k % 4)
        for e in range(3): tt.span(g, 3, ks + 2 + 3 * e, ks + 4 + 3 * e, (k + e) % 4)
        if k % 40 == 0: tt.span(g, 2, tl, tl + 40 * 300, k % 4)
        if k % 5 == 0:
            tt.ev(g, tl, ks + d // 3, ks + d + 500, kind=AG if k % 10 else RS, stream=1 + (k % 10 == 0), name=3); names.append(3)
        tt.sample(g, ks + d // 2, int(rng.integers(1300, 2100)), int(rng.integers(500, 900)))
        t = ks + d + int(rng.integers(5, 60))
    tt.counter_pass(g, names, [0, 1], rng.integers(0, 1000, size=(2, len(names))).astype(float))
b = tt.bundle()
p = params(b, f_gemm=np.full(4, 1e9), op_type=np.array([1, 2, 0, 1], np.int32))
ref, got, res, _ = run_both(b, p)
a = ref['inst.counters'].reshape(2, -1); c = got['inst.counters'].reshape(2, -1)
bad = np.nonzero(~np.isclose(a, c, rtol=1e-9).all(0))[0]
print("N", b.n_events, "rows", a.shape[1], "bad rows", len(bad), bad[:10])
for j in bad[:6]:
    print(j, ref['inst.gpu'][j], ref['inst.first_idx'][j], ref['inst.n_events'][j], a[:, j], c[:, j])
