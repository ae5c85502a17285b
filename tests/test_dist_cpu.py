"""Multi-process (world_size 2, gloo, CPU) tests of the output-channel sharding host logic in
paper_2506_11586_b200/dist.py: slicing, the padded all-gather layout and the reassembly of the
server's output shares. The per-rank shares are computed here with the oracle's index map
(a stand-in for secn_extract_share, which needs a GPU); the collective and the bookkeeping are
exactly what bench.py runs on NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_11586_b200 import dist as sdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_m_slices_cover_and_balance():
    for M in (1, 7, 16, 64, 1000, 1001):
        for world in (1, 2, 3, 4, 8):
            sl = sdist.m_slices(M, world)
            assert len(sl) == world
            assert sl[0][0] == 0 and sum(mc for _, mc in sl) == M
            for (a, ma), (b, _) in zip(sl, sl[1:]):
                assert a + ma == b
            sizes = [mc for _, mc in sl]
            assert max(sizes) - min(sizes) <= 1
            assert max(sizes) <= sdist.padded_slice(M, world)


def _worker(rank, world, port, dims, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        layout = sdist.share_layout(dims, world)
        local = torch.zeros(layout.chunk, dtype=torch.int64)
        for (M, OH, OW), off in zip(dims, layout.offsets):
            m0, mc = sdist.m_slices(M, world)[rank]
            # each rank fills its slice with a value that encodes the global (m, oy, ox)
            m = torch.arange(m0, m0 + mc).view(-1, 1, 1)
            val = (m * 1_000_000 + torch.arange(OH).view(1, -1, 1) * 1000 + torch.arange(OW).view(1, 1, -1))
            local[off:off + mc * OH * OW] = val.reshape(-1)
        gathered = sdist.all_gather_shares(local, world)
        full = sdist.reassemble(gathered, layout, dims, world)
        ok = True
        for (M, OH, OW), f in zip(dims, full):
            ref = (torch.arange(M).view(-1, 1, 1) * 1_000_000 + torch.arange(OH).view(1, -1, 1) * 1000
                   + torch.arange(OW).view(1, 1, -1))
            ok &= f.shape == (M, OH, OW) and bool(torch.equal(f, ref))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_all_gather_reassembles_every_layer(world):
    dims = [(64, 111, 111), (16, 55, 55), (1000, 13, 13), (7, 3, 5)]  # includes M not divisible by world
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, dims, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert sorted(r for r, _ in res) == list(range(world))
    assert all(ok for _, ok in res)


def _plan_worker(rank, world, port, q):
    """Every rank derives the same full-M plan, and the union of the rank-local output-channel
    slices equals the layer's output channels (what bench.py relies on)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import packing
        from workloads import layers

        ok = True
        for l in layers.squeezenet11():
            p = packing.plan_conv(l.C, l.H, l.W, l.M, l.k, l.k, l.stride, l.pad, 4096, 2, rule="time")
            t = torch.tensor([p.Cw, p.Hw, p.Ww, p.G, p.S, p.O], dtype=torch.int64)
            ts = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(ts, t)
            ok &= all(torch.equal(ts[0], x) for x in ts)
            m0, mc = sdist.m_slices(l.M, world)[rank]
            cnt = torch.tensor([mc], dtype=torch.int64)
            dist.all_reduce(cnt)
            ok &= int(cnt) == l.M
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_ranks_agree_on_plans_and_cover_channels():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_plan_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(ok for _, ok in res)


def test_partition_covers_every_output_once():
    from oracle import packing
    from workloads import layers

    for world in (1, 2, 3, 4, 8):
        for M, S in [(16, 4), (1, 1), (3, 7), (64, 1), (1000, 1), (5, 16), (16, 2), (32, 2)]:
            parts = sdist.partition(M, S, world)
            assert len(parts) == world
            seen = np.zeros((M, S), np.int32)
            for p in parts:
                seen[p.m0:p.m0 + p.mc, p.s0:p.s0 + p.sc] += 1
            assert (seen == 1).all(), (M, S, world)
    # the grid goes spatial only where channel slices would be thinner than an m-block
    assert len({(p.s0, p.sc) for p in sdist.partition(16, 4, 8)}) > 1
    for l in layers.resnet50():
        p = packing.plan_conv(l.C, l.H, l.W, l.M, l.k, l.k, l.stride, l.pad, 4096, 2, rule="time")
        assert all(x.sc == p.S for x in sdist.partition(l.M, p.S, 8)), l.name


def test_block_of_output_matches_oracle_designation():
    from oracle import packing
    from workloads import layers

    class Pl:  # the fields block_of_output reads, from the oracle's plan
        def __init__(self, o):
            for f in ("OH", "OW", "Hw", "Ww", "kh", "kw", "stride", "decim", "nbw"):
                setattr(self, f, getattr(o, f))

    for l in layers.squeezenet11()[:4] + [layers.ConvLayer("s2", 3, 40, 40, 5, 3, 2, 0),
                                          layers.ConvLayer("ds", 24, 28, 28, 9, 1, 2, 0)]:
        for rule in ("time", "bytes"):
            o = packing.plan_conv(l.C, l.H, l.W, l.M, l.k, l.k, l.stride, l.pad, 4096, 2, rule=rule)
            s_idx, _ = packing.designated_map(o)
            assert (sdist.block_of_output(Pl(o)).numpy() == s_idx).all(), (l.name, rule)


def _part_worker(rank, world, port, q):
    """The (channel x spatial block) partition end to end on gloo: each rank fills the shares it
    owns (a value encoding (m, oy, ox)) into its chunk -- and garbage at positions it does not own
    -- all-gathers, and reassembles with the owner map."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import packing

        geo = [(16, 55, 55, 1, 1, 1, 0, 64), (64, 224, 224, 3, 3, 2, 0, 3), (7, 13, 13, 3, 3, 1, 1, 5)]
        plans, dims, parts, blocks = [], [], [], []
        for M, H, W, k, _, st, pad, C in geo:
            o = packing.plan_conv(C, H, W, M, k, k, st, pad, 4096, 2, rule="time")
            plans.append(o)
            dims.append((M, o.OH, o.OW))
            parts.append(sdist.partition(M, o.S, world, mblock=16))
            s_idx, _ = packing.designated_map(o)
            blocks.append(torch.from_numpy(s_idx))
        layout = sdist.share_layout(dims, world, parts)
        local = torch.full((layout.chunk,), -7, dtype=torch.int64)
        for (M, OH, OW), off, pt, b in zip(dims, layout.offsets, parts, blocks):
            p = pt[rank]
            m = torch.arange(p.m0, p.m0 + p.mc).view(-1, 1, 1)
            val = m * 1_000_000 + torch.arange(OH).view(1, -1, 1) * 1000 + torch.arange(OW).view(1, 1, -1)
            own = (b >= p.s0) & (b < p.s0 + p.sc)
            val = torch.where(own, val, torch.full_like(val, -1))  # positions of other ranks: garbage
            local[off:off + p.mc * OH * OW] = val.reshape(-1)
        full = sdist.reassemble(sdist.all_gather_shares(local, world), layout, dims, world, parts, blocks)
        ok = True
        for (M, OH, OW), f in zip(dims, full):
            ref = (torch.arange(M).view(-1, 1, 1) * 1_000_000 + torch.arange(OH).view(1, -1, 1) * 1000
                   + torch.arange(OW).view(1, 1, -1))
            ok &= bool(torch.equal(f, ref))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_partition_all_gather_reassembles():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_part_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(ok for _, ok in res)
