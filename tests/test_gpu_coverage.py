"""GPU parity on the configurations round 1 left untested ("Untested configurations"):
every SqueezeNet-1.0 and ResNet-50 layer at full size, the accumulator's worst case at the
kernel's G limit, rank-sliced calls reassembled as the multi-GPU path does, and the CUDA
sanitizers. Every comparison is word for word against the oracle (or a closed form).

Run on a B200 with: python -m pytest tests -m gpu
"""
import os
import shutil
import subprocess
import sys
import zlib
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import he, packing, philox
from test_gpu_parity import DEV, TP, UP, Dev, _layer_inputs, env, oplan, secn, secn_mod  # noqa: F401  (fixtures)
from workloads import layers

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _check_layer(ctx, P, D, lay, seed, n_samples):
    """Runs the whole layer on the GPU (bench launch configuration) and compares whole output
    ciphertexts -- the first, the last and n_samples random ones -- and every word of the fused
    server share y0 with the oracle."""
    opl = oplan(P, ctx, lay)
    ct, x0, K, r = _layer_inputs(P, lay, seed, opl)
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    w = ctx.preprocess_weights(plan, TP(K))
    y0 = torch.full((plan.M, plan.OH, plan.OW), -1, dtype=torch.int64, device=DEV)
    got = D.U(ctx.he_conv2d(plan, D.R(ct), w, x0=TP(x0), r=TP(r), y0=y0))
    n_out = opl.M * opl.S
    g = np.random.default_rng(seed + 1)
    pick = np.unique(np.concatenate([[0, n_out - 1], g.integers(0, n_out, n_samples)]))
    sel = np.zeros(n_out, np.uint8)
    sel[pick] = 1
    ref = he.server_conv(ct, x0, K, r, opl, P, sel=sel)
    assert (got[pick] == ref[pick]).all(), lay.name
    assert (UP(y0) == packing.extract((P.t - r) % P.t, opl)).all(), lay.name


@pytest.mark.parametrize("lay", layers.squeezenet10(), ids=lambda l: l.name)
def test_squeezenet10_every_layer_full_size(env, lay):
    """All 26 SqueezeNet-1.0 layers (conv1 is 3 -> 96, 7x7 / 2: BASELINE.json configs[1])."""
    ctx, P, D = env
    _check_layer(ctx, P, D, lay, 500 + zlib.crc32(lay.name.encode()) % 1000, 2)


@pytest.mark.parametrize("lay", layers.resnet50(), ids=lambda l: l.name)
def test_resnet50_every_layer_full_size(env, lay):
    """All 53 ResNet-50 v1.5 conv layers (BASELINE.json configs[3]), including the G = 29/30
    windows of the 1024/2048-channel layers."""
    ctx, P, D = env
    _check_layer(ctx, P, D, lay, 700 + zlib.crc32(lay.name.encode()) % 1000, 1)


def test_resnet50_plans_reach_g29(env):
    ctx, P, D = env
    assert max(oplan(P, ctx, l).G for l in layers.resnet50()) >= 29


@pytest.mark.parametrize("m", [1, 3])
def test_mac_worst_case_accumulator_g32(env, m):
    """The MAC's worst case at the kernel's limit G = 32 (explicit 64 x 64 window: Cw = 1): every
    NTT-domain input word and every NTT-domain weight word is q_j - 1 (the largest residue), the
    mask is t - 1. 32-bit limbs: 32 (q-1)^2 < q 2^32 is the lazy-sum / REDC precondition; 64-bit
    limbs: 32 products < 2^122 in the 128-bit sum. Closed form: sum_g (q-1)^2 = G mod q in every
    NTT slot, and the inverse NTT of a constant vector c is the constant polynomial c (checked
    also with the oracle's direct inverse NTT); b then gains enc(t - 1)."""
    ctx, P, D = env
    G = 32
    lay = layers.ConvLayer("g32", G, 64, 64, m, 1, 1, 0)
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, 1, Hw=64, Ww=64)
    assert (plan.G, plan.S, plan.Cw) == (G, 1, 1)
    L, n = ctx.L, ctx.n
    qmax = np.array([q - 1 for q in P.primes], np.uint64)
    xh = np.broadcast_to(qmax[None, None, :, None], (G, 2, L, n)).copy()
    wn = np.broadcast_to(qmax[None, None, :, None], (m, G, L, n)).copy()
    r = np.full((m, n), P.t - 1, np.uint64)
    ws = torch.empty(ctx.workspace_bytes(plan) // 8, dtype=torch.int64, device=DEV)
    wsv = ws.view(ctx.rdtype)[: G * 2 * L * n].view(G, 2, L, n)
    wsv.copy_(D.R(xh))
    out = ctx.empty(m, 2, L, n)
    ct_dummy = ctx.empty(G, 2, L, n)
    w = D.R(wn)
    rt = TP(r)
    ctx.he_conv2d_stage(1, plan, ct_dummy, w, None, rt, out, ws)
    ctx.he_conv2d_stage(2, plan, ct_dummy, w, None, rt, out, ws)
    got = D.U(out)
    for j, q in enumerate(P.primes):
        c = G % q
        flat = np.zeros(n, np.uint64)
        flat[0] = c
        assert (he.intt(np.full(n, c, np.uint64), P, j) == flat).all()  # the oracle agrees with the closed form
        enc_r = he.enc(np.full(n, P.t - 1, np.uint64), P, j)
        exp_b = (flat.astype(object) + enc_r.astype(object)) % q
        for mm in range(m):
            assert (got[mm, 0, j] == flat).all(), (mm, j)
            assert (got[mm, 1, j] == exp_b.astype(np.uint64)).all(), (mm, j)


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("name", ["fire9.e3", "conv1", "fire2.sq", "fire3.sq"])
@pytest.mark.parametrize("drawn", [False, True], ids=["r_in", "r_drawn"])
def test_rank_partition_calls_reassemble(env, world, name, drawn):
    """Each rank's call of the multi-GPU path (bench.py: dist.partition's (channel x spatial
    block) rectangle -> plan.copy(M=mc, s_begin, s_count), the rank's weights, mask rows -- given,
    or drawn with ct0 = m0 S -- and share block), run one after another on this GPU, then
    reassembled with dist.reassemble exactly as after the NCCL all-gather: every output ciphertext
    (from the rank that owns it) and every server share equal the oracle's single-GPU result.
    fire2.sq / fire3.sq at 4 and 8 ranks take spatial slices (Ps > 1)."""
    from paper_2506_11586_b200 import dist as sdist

    ctx, P, D = env
    lay = next(l for l in layers.squeezenet11() if l.name == name)
    opl = oplan(P, ctx, lay)
    ct, x0, K, r = _layer_inputs(P, lay, 900 + world, opl)
    seed, stream = 31337, 4
    if drawn:
        r = philox.mask(seed, stream, opl.M * opl.S, P.n, P.t_bits)
    plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    S = plan.S
    parts = sdist.partition(plan.M, S, world)
    dims = [(plan.M, plan.OH, plan.OW)]
    layout = sdist.share_layout(dims, world, [parts])
    chunks = []
    got = np.zeros((plan.M * S, 2, ctx.L, ctx.n), np.uint64)
    owned = np.zeros(plan.M * S, bool)
    cti, x0t = D.R(ct), TP(x0)
    for p in parts:
        chunk = torch.full((layout.chunk,), -5, dtype=torch.int64, device=DEV)
        if p.mc > 0:
            sl = p.sc < S
            pl = plan.copy(M=p.mc, s_begin=p.s0 if sl else 0, s_count=p.sc if sl else 0)
            w = ctx.preprocess_weights(pl, TP(np.ascontiguousarray(K[p.m0:p.m0 + p.mc])))
            y0 = chunk[layout.offsets[0]:layout.offsets[0] + p.mc * plan.OH * plan.OW].view(p.mc, plan.OH, plan.OW)
            if drawn:
                g = secn_mod().MaskGen(seed=seed, stream=stream, ct0=p.m0 * S)
                o = D.U(ctx.he_conv2d_gen(pl, cti, w, g, x0=x0t, y0=y0))
            else:
                o = D.U(ctx.he_conv2d(pl, cti, w, x0=x0t, r=TP(np.ascontiguousarray(r[p.m0 * S:(p.m0 + p.mc) * S])),
                                      y0=y0))
            for m in range(p.mc):
                for s_ in range(p.s0, p.s0 + p.sc):
                    row = (p.m0 + m) * S + s_
                    assert not owned[row]
                    owned[row] = True
                    got[row] = o[m * S + s_]
        chunks.append(chunk)
    assert owned.all()
    full = sdist.reassemble(torch.cat(chunks), layout, dims, world, [parts], [sdist.block_of_output(plan)])[0]
    n_out = opl.M * opl.S
    pick = np.unique(np.array([0, n_out // 3, n_out // 2, n_out - 1, min(n_out - 1, S)]))
    sel = np.zeros(n_out, np.uint8)
    sel[pick] = 1
    ref = he.server_conv(ct, x0, K, r, opl, P, sel=sel)
    assert (got[pick] == ref[pick]).all()
    assert (UP(full) == packing.extract((P.t - r) % P.t, opl)).all()


SANITIZER = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"

_SAN_LAYER = """
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import __graft_entry__ as g
g.build()
from paper_2506_11586_b200 import Context
from workloads import inputs, layers
ctx = Context(0, word_bits={wb})
lay = [l for l in layers.squeezenet11() if l.name == {name!r}][0]
plan = ctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
gen = inputs.rng(3)
ct = inputs.uniform_residues(gen, (plan.G * plan.S, 2), ctx.primes, ctx.n)
R = (lambda a: torch.from_numpy(a.view(np.int64)).cuda()) if {wb} == 64 else \\
    (lambda a: torch.from_numpy(a.astype(np.uint32).view(np.int32)).cuda())
T = lambda a: torch.from_numpy(a.view(np.int64)).cuda()
x0 = inputs.uniform_below(gen, (plan.G * plan.S, ctx.n), 1 << 37)
K = inputs.quantized_kernel(gen, plan.M, lay.C, lay.k, lay.k)
r = inputs.uniform_below(gen, (plan.M * plan.S, ctx.n), 1 << 37)
w = ctx.preprocess_weights(plan, T(K))
y0 = torch.empty((plan.M, plan.OH, plan.OW), dtype=torch.int64, device='cuda')
out = ctx.he_conv2d(plan, R(ct), w, x0=T(x0), r=T(r), y0=y0)
torch.cuda.synchronize()
print('SANITIZED_RUN_OK')
"""


def _sanitize(tool, code, timeout=900):
    if not Path(SANITIZER).exists():
        pytest.skip("compute-sanitizer not installed")
    res = subprocess.run([SANITIZER, f"--tool={tool}", "--error-exitcode=97", "--print-limit=20",
                          sys.executable, "-c", code], capture_output=True, text=True, timeout=timeout, cwd=ROOT,
                         env={**os.environ, "PYTHONPATH": str(ROOT)})
    tail = (res.stdout[-3000:] + res.stderr[-3000:])
    if "compute-sanitizer is closed on this pool" in tail:  # the GPU pool's wrapper refuses it (leaves GPUs needing a reset)
        pytest.skip("compute-sanitizer is disabled on this GPU pool: " + tail.strip().splitlines()[0][:200])
    assert res.returncode == 0, f"{tool}: rc={res.returncode}\n{tail}"
    assert "SANITIZED_RUN_OK" in res.stdout or "smoke OK" in res.stdout, tail
    assert "ERROR SUMMARY: 0 errors" in res.stdout + res.stderr or "RACECHECK SUMMARY: 0 hazards" in res.stdout + res.stderr, tail


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_sanitizer_smoke(tool):
    """compute-sanitizer over smoke(): the tiny config through every hot-path kernel."""
    _sanitize(tool, f"import sys; sys.path.insert(0, {str(ROOT)!r}); import __graft_entry__ as g; g.smoke()")


@pytest.mark.parametrize("wb", [32, 64])
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_conv1_layer(tool, wb):
    """compute-sanitizer over a full SqueezeNet-1.1 conv1 layer (polyphase plan, S > 1, several
    m-blocks per CTA) and a fire squeeze layer."""
    for name in ("conv1", "fire3.sq"):
        _sanitize(tool, _SAN_LAYER.format(root=str(ROOT), wb=wb, name=name), timeout=1500)


@pytest.mark.parametrize("sgmt", ["1,1", "1,2", "1,4", "2,1", "2,2"])
@pytest.mark.parametrize("name", ["fire9.e3", "conv1", "fire3.sq", "fire6.sq"])
def test_fused_layer_kernel_exact(env, sgmt, name, monkeypatch):
    """The fused small-layer kernel (k_layer_fused: MAC + all 12 inverse-NTT levels + mask + share
    in one launch; SECN_FUSED=2, off by default) in every register block, exact against the
    oracle on S > 1 (conv1: polyphase, ragged s-groups), large-G and many-m-block layers."""
    ctx, P, D = env
    if ctx.word_bits != 32:
        pytest.skip("32-bit limbs only")
    sg, mt = sgmt.split(",")
    monkeypatch.setenv("SECN_FUSED", "2")
    monkeypatch.setenv("SECN_FUSED_SG", sg)
    monkeypatch.setenv("SECN_FUSED_MT", mt)
    fctx = secn_mod().Context(0, word_bits=32)
    lay = next(l for l in layers.squeezenet11() if l.name == name)
    opl = oplan(P, fctx, lay)
    ct, x0, K, r = _layer_inputs(P, lay, 77, opl)
    plan = fctx.plan(lay.C, lay.H, lay.W, lay.M, lay.k, stride=lay.stride, pad=lay.pad)
    w = fctx.preprocess_weights(plan, TP(K))
    y0 = torch.full((plan.M, plan.OH, plan.OW), -1, dtype=torch.int64, device=DEV)
    got = D.U(fctx.he_conv2d(plan, D.R(ct), w, x0=TP(x0), r=TP(r), y0=y0))
    fctx.close()
    n_out = opl.M * opl.S
    pick = np.unique(np.array([0, 1, n_out // 2, n_out - 1]))
    sel = np.zeros(n_out, np.uint8)
    sel[pick] = 1
    ref = he.server_conv(ct, x0, K, r, opl, P, sel=sel)
    assert (got[pick] == ref[pick]).all()
    assert (UP(y0) == packing.extract((P.t - r) % P.t, opl)).all()
