"""C-ABI library checks that need no GPU: it loads, exports every symbol include/secn.h
declares, its host-only plan call agrees with the oracle's plan rule on every layer of the
paper's workloads, and its error paths return status codes instead of crashing."""
import ctypes
import re
from pathlib import Path

import pytest

import __graft_entry__
from oracle import packing
from workloads import layers

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def secn():
    __graft_entry__.build()
    from paper_2506_11586_b200 import secn as m

    return m


def _header_functions():
    text = (ROOT / "include" / "secn.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(secn(?:32)?_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(secn):
    names = _header_functions()
    assert len(names) >= 12
    lib = secn.lib()
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(secn.EXPORTS)


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(ROOT / "paper_2506_11586_b200" / "libsecn.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if ".cubin" in line)


@pytest.mark.parametrize("net", ["tiny", "squeezenet1_1", "squeezenet1_0", "resnet50"])
def test_c_plan_matches_oracle_plan(secn, net):
    fields = ("OH", "OW", "decim", "Hp", "Wp", "Cw", "Hw", "Ww", "G", "S", "nbh", "nbw", "O")
    for l in layers.network(net):
        c = secn.conv_plan(l.C, l.H, l.W, l.M, l.k, stride=l.stride, pad=l.pad, rule=secn.PLAN_BYTES)
        o = packing.plan_conv(l.C, l.H, l.W, l.M, l.k, l.k, l.stride, l.pad, 4096, 2)
        assert tuple(getattr(c, f) for f in fields) == tuple(getattr(o, f) for f in fields), l.name


def test_c_plan_other_ring_sizes_and_explicit_windows(secn):
    for l in [layers.ConvLayer("a", 64, 56, 56, 64, 3, 1, 1), layers.ConvLayer("b", 3, 224, 224, 64, 7, 2, 3)]:
        for logn, L in [(13, 2), (14, 4)]:
            c = secn.conv_plan(l.C, l.H, l.W, l.M, l.k, stride=l.stride, pad=l.pad, log_n=logn, n_limbs=L,
                               rule=secn.PLAN_BYTES)
            o = packing.plan_conv(l.C, l.H, l.W, l.M, l.k, l.k, l.stride, l.pad, 1 << logn, L)
            assert (c.Cw, c.Hw, c.Ww, c.G, c.S, c.O) == (o.Cw, o.Hw, o.Ww, o.G, o.S, o.O)
    c = secn.conv_plan(8, 16, 16, 3, 3, pad=1, Hw=10, Ww=9)
    o = packing.plan_conv(8, 16, 16, 3, 3, 3, 1, 1, 4096, 2, Hw=10, Ww=9)
    assert (c.Cw, c.G, c.S, c.nbh, c.nbw, c.O) == (o.Cw, o.G, o.S, o.nbh, o.nbw, o.O)


@pytest.mark.parametrize("net", ["tiny", "squeezenet1_1", "squeezenet1_0", "resnet50"])
def test_c_time_plan_matches_oracle_time_rule(secn, net):
    """The default plan (reading R6b): the library's window equals the oracle's
    plan_conv(rule="time") on every layer, G <= 32, and it is never modelled slower than the
    byte-min plan. The tests, smoke() and bench.py take the window from the oracle and assert this
    equality, so no oracle input depends on the product library."""
    fields = ("OH", "OW", "decim", "Hp", "Wp", "Cw", "Hw", "Ww", "G", "S", "nbh", "nbw", "O")
    for l in layers.network(net):
        c = secn.conv_plan(l.C, l.H, l.W, l.M, l.k, stride=l.stride, pad=l.pad)
        o = packing.plan_conv(l.C, l.H, l.W, l.M, l.k, l.k, l.stride, l.pad, 4096, 2, rule="time")
        assert tuple(getattr(c, f) for f in fields) == tuple(getattr(o, f) for f in fields), l.name
        assert c.G <= 32


@pytest.mark.parametrize("logn,cw", [(12, 1), (12, 4), (13, 2), (14, 2)])
def test_c_time_plan_matches_oracle_other_rings(secn, logn, cw):
    fields = ("decim", "Cw", "Hw", "Ww", "G", "S", "O")
    for l in layers.squeezenet11()[:6] + [layers.ConvLayer("s2", 32, 30, 30, 40, 5, 2, 2)]:
        c = secn.conv_plan(l.C, l.H, l.W, l.M, l.k, stride=l.stride, pad=l.pad, log_n=logn, n_limbs=cw)
        o = packing.plan_conv(l.C, l.H, l.W, l.M, l.k, l.k, l.stride, l.pad, 1 << logn, cw, rule="time")
        assert tuple(getattr(c, f) for f in fields) == tuple(getattr(o, f) for f in fields), (l.name, logn, cw)


@pytest.mark.parametrize("n_i,n_o,logn,cw", [(2048, 1000, 12, 2), (512, 1000, 12, 2), (64, 16, 12, 2), (4096, 1, 12, 1),
                                             (1, 4096, 12, 2), (100, 37, 8, 2), (2048, 1000, 13, 2), (9216, 4096, 14, 4)])
def test_c_fc_plan_matches_oracle_plan(secn, n_i, n_o, logn, cw):
    from oracle import fc

    c = secn.fc_plan(n_i, n_o, log_n=logn, coef_words64=cw)
    o = fc.plan_fc(n_i, n_o, 1 << logn, cw)
    assert (c.nib, c.nob, c.G, c.M) == (o.nib, o.nob, o.G, o.M)
    c2 = secn.fc_plan(n_i, n_o, log_n=logn, coef_words64=cw, nib=max(1, o.nib // 2))
    o2 = fc.plan_fc(n_i, n_o, 1 << logn, cw, nib=max(1, o.nib // 2))
    assert (c2.nib, c2.nob, c2.G, c2.M) == (o2.nib, o2.nob, o2.G, o2.M)


def test_c_fc_plan_errors(secn):
    for args in [(0, 5), (5, 0)]:
        with pytest.raises(secn.SecnError) as e:
            secn.fc_plan(*args)
        assert e.value.status == -1
    with pytest.raises(secn.SecnError):
        secn.fc_plan(10, 10, nib=11)


def test_error_paths_return_status(secn):
    lib = secn.lib()
    with pytest.raises(secn.SecnError) as e:
        secn.conv_plan(4, 2, 2, 8, 3)  # kernel larger than the input
    assert e.value.status == -2
    with pytest.raises(secn.SecnError) as e:
        secn.conv_plan(4, 16, 16, 8, 3, Hw=100, Ww=100)  # explicit window larger than N
    assert e.value.status == -1
    h = ctypes.c_void_p()
    bad = (ctypes.c_uint64 * 1)(12289)  # = 1 mod 8192? no: 12289 = 3*4096 + 1, not = 1 mod 8192
    assert lib.secn_ctx_create(ctypes.byref(h), 0, 12, 1, bad, 37) == -2
    big = (ctypes.c_uint64 * 1)((1 << 62) - 57)
    assert lib.secn_ctx_create(ctypes.byref(h), 0, 12, 1, big, 37) == -2
    assert lib.secn_ctx_create(ctypes.byref(h), 0, 11, 1, bad, 37) == -2
    assert lib.secn_ctx_create(None, 0, 12, 1, bad, 37) == -1
    assert lib.secn_ntt_fwd(None, None, 0, None) == -1
    assert b"NULL" in lib.secn_last_error()
