"""CPU-side checks of the boundary: the C-ABI library builds, loads without a GPU and exports every
symbol include/chopper.h declares; host argument checks fail loudly; the product path has no CPU fallback."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import paper_2512_08242_b200 as ch
    ch.build()
    return ch.load_library()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "chopper.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(chopper_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    import paper_2512_08242_b200 as ch
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(ch.EXPORTS) == syms


def test_abi_version_and_scratch(lib):
    import paper_2512_08242_b200 as ch
    assert lib.chopper_abi_version() == 8
    cfg = ch.chopper_config(n_traced_gpus=8, n_labels=42, max_iters=256, max_coll_per_class=20000)
    small = ch.chopper_scratch_bytes(cfg, 1000, 100, 0, 0)
    big = ch.chopper_scratch_bytes(cfg, 20_000_000, 2_000_000, 1_000_000, 8)
    assert 0 < small < big


def test_create_rejects_bad_args(lib):
    import ctypes

    import paper_2512_08242_b200 as ch
    ctx = ctypes.c_void_p()
    cfg = ch.chopper_config(n_traced_gpus=0, n_labels=1, max_iters=1, max_coll_per_class=1)
    buf = ctypes.create_string_buffer(16)
    assert lib.chopper_create(ctypes.byref(ctx), ctypes.byref(cfg), 0, None, None, 0, 1,
                              ctypes.cast(buf, ctypes.c_void_p), 16) == 2
    cfg.n_traced_gpus = 2
    # rank outside 0..nranks-1
    assert lib.chopper_create(ctypes.byref(ctx), ctypes.byref(cfg), 0, None, None, 2, 2,
                              ctypes.cast(buf, ctypes.c_void_p), 16) == 2


def test_loopback_group_sizes(lib):
    """the in-process transport's group accepts 1..256 ranks (host logic; the copy itself needs a GPU)"""
    assert not lib.chopper_loopback_create(0) and not lib.chopper_loopback_create(257)
    g = lib.chopper_loopback_create(4)
    assert g
    # a rank outside the group is refused before touching the device
    assert lib.chopper_loopback_allgather(g, None, None, 8, 4, 4, None) != 0
    assert lib.chopper_loopback_allgather(g, None, None, 8, 0, 3, None) != 0
    lib.chopper_loopback_destroy(g)


def test_no_cpu_fallback():
    import torch

    import paper_2512_08242_b200 as ch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        ch.Pipeline(2, 4, 4, 4)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2512_08242_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import|from)\s+(oracle|tracegen)\b", txt, flags=re.M), f
                assert "chopper_oracle" not in txt and "libchopper_oracle" not in txt, f
                assert "oracle_run" not in txt and "or_run" not in txt, f


def test_flops_table_spec_examples(golden):
    """host F_gemm table of the product side (Eq. 4): SPEC.md:354-355 examples and scaling."""
    import paper_2512_08242_b200 as ch
    g = golden("breakdown.json")["flops"]
    one = dict(b=1, s=2, hidden=2, ffn=2, heads=1, kv_heads=1, head_dim=2, vocab=2, layers=1)
    t = ch.flops_table(["f_attn_fa", "f_attn_op"], one)
    assert t[0] == g["attn"]           # 4*b*h*s^2*d
    assert t[1] == 2 * 2 * 2 * 2       # m = b*s = 2, n = k = hidden = 2
