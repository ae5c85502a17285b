"""Multi-GPU sharding of the HE convolution by output channel and spatial block.

One process per GPU. Every rank holds the same input ciphertexts (the client's upload is
broadcast once) and the same layer plan (computed for the FULL output-channel count M, so the
packing of the inputs does not depend on the number of ranks). The M x S output ciphertexts of a
layer are split into a Pm x Ps grid of rectangles (`partition`): rank k owns the channels
[m0, m0 + mc) and the spatial blocks [s0, s0 + sc); it preprocesses only those channels' weights
and runs secn_he_conv2d on a plan copy with M = mc and the spatial slice (s_begin, s_count). For
the SqueezeNet / ResNet-50 shapes the grid is Ps = 1 (contiguous channel slices) except where
the slices would be thinner than the MAC kernel's m-block.
The only collective is an all-gather of those shares (the north star's "NCCL all-gather over
NVLink only to collect output shares"); output ciphertexts stay on the rank that computed them.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Tuple

import torch
import torch.distributed as dist


def m_slices(M: int, world: int) -> List[Tuple[int, int]]:
    """Balanced contiguous slices: the first M % world ranks get one extra channel."""
    base, extra = divmod(M, world)
    out, m0 = [], 0
    for k in range(world):
        mc = base + (1 if k < extra else 0)
        out.append((m0, mc))
        m0 += mc
    return out


@dataclass(frozen=True)
class Part:
    """One rank's share of a layer's output: channels [m0, m0 + mc) x spatial blocks [s0, s0 + sc)."""
    m0: int
    mc: int
    s0: int
    sc: int


def _slices(n: int, k: int) -> List[Tuple[int, int]]:
    base, extra = divmod(n, k)
    out, a = [], 0
    for i in range(k):
        c = base + (1 if i < extra else 0)
        out.append((a, c))
        a += c
    return out


def partition(M: int, S: int, world: int, mblock: int = 8) -> List[Part]:
    """The (m, s) partition of one layer's M x S output ciphertexts: the ranks form
    a Pm x Ps grid (Ps a divisor of world, Ps <= S) and rank im * Ps + is owns the im-th contiguous
    channel slice and the is-th contiguous block slice. Ps > 1 only pays where the channel slices
    alone would be thin: the MAC kernel computes whole m-blocks of `mblock` channels, so a rank's
    work is modelled as ceil(mc / mblock) * mblock * sc padded output ciphertexts; the grid with the
    smallest largest-rank work wins (ties: fewer s-slices, which keeps the weights of an output
    channel on one rank)."""
    best = None
    for ps in range(1, world + 1):
        if world % ps or ps > S:
            continue
        pm = world // ps
        ms, ss = _slices(M, pm), _slices(S, ps)
        work = max(-(-mc // mblock) * mblock * sc for _, mc in ms for _, sc in ss)
        if best is None or work < best[0]:
            best = (work, ms, ss)
    _, ms, ss = best
    return [Part(m0, mc, s0, sc) for m0, mc in ms for s0, sc in ss]


def block_of_output(plan) -> "torch.Tensor":
    """s[oy, ox]: the spatial block (output ciphertext column) holding output (oy, ox) under the
    plan's designation (include/secn.h: (bh (Hw-kh+1) + i, bw (Ww-kw+1) + j) = (oy sh, ox sh),
    with the phase-split kernel extent for polyphase plans)."""
    ps = plan.stride if plan.decim == 2 else 1
    khe, kwe = -(-plan.kh // ps), -(-plan.kw // ps)
    sh = 1 if plan.decim else plan.stride
    oy = torch.arange(plan.OH).view(-1, 1) * sh
    ox = torch.arange(plan.OW).view(1, -1) * sh
    return (oy // (plan.Hw - khe + 1)) * plan.nbw + ox // (plan.Ww - kwe + 1)


def padded_slice(M: int, world: int) -> int:
    """Rows per rank in the all-gather buffer (all-gather needs equal sizes)."""
    return -(-M // world)


@dataclass
class ShareLayout:
    """Where each layer's share block lives in one flat per-step all-gather buffer."""
    offsets: List[int]       # per layer, offset (elements) within a rank's chunk
    sizes: List[int]         # per layer, padded rows * OH * OW
    chunk: int               # elements per rank


def share_layout(dims: List[Tuple[int, int, int]], world: int, parts: Optional[List[List[Part]]] = None
                 ) -> ShareLayout:
    """dims = [(M, OH, OW)] per layer; parts = the per-layer partitions (default: channel slices).
    A rank's chunk holds, per layer, its channel rows [max mc][OH][OW] (the positions of other
    ranks' spatial blocks in it are ignored by reassemble)."""
    offs, sizes, o = [], [], 0
    for li, (M, OH, OW) in enumerate(dims):
        rows = max(p.mc for p in parts[li]) if parts is not None else padded_slice(M, world)
        sz = rows * OH * OW
        offs.append(o)
        sizes.append(sz)
        o += sz
    return ShareLayout(offs, sizes, o)


def reassemble(gathered: torch.Tensor, layout: ShareLayout, dims: List[Tuple[int, int, int]], world: int,
               parts: Optional[List[List[Part]]] = None, blocks: Optional[List[torch.Tensor]] = None
               ) -> List[torch.Tensor]:
    """gathered [world * chunk] -> per layer full share tensor [M, OH, OW]: rank k's rows are
    channels [m0, m0 + mc); with spatial slices (sc < S) only the outputs whose block s
    (blocks[layer][oy, ox], see block_of_output) lies in [s0, s0 + sc) come from rank k."""
    g = gathered.view(world, layout.chunk)
    out = []
    for li, ((M, OH, OW), off, sz) in enumerate(zip(dims, layout.offsets, layout.sizes)):
        if parts is None:
            rows = padded_slice(M, world)
            out.append(torch.cat([g[k, off:off + sz].view(rows, OH, OW)[:mc]
                                  for k, (m0, mc) in enumerate(m_slices(M, world))], 0))
            continue
        rows = sz // (OH * OW)
        full = torch.zeros((M, OH, OW), dtype=gathered.dtype, device=gathered.device)
        for k, p in enumerate(parts[li]):
            blk = g[k, off:off + sz].view(rows, OH, OW)[:p.mc]
            if blocks is None:
                full[p.m0:p.m0 + p.mc] = blk
            else:
                own = ((blocks[li] >= p.s0) & (blocks[li] < p.s0 + p.sc)).to(gathered.device)
                full[p.m0:p.m0 + p.mc] = torch.where(own, blk, full[p.m0:p.m0 + p.mc])
        out.append(full)
    return out


def all_gather_shares(local: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """local [chunk] -> [world * chunk] via one all_gather_into_tensor (NCCL on GPUs)."""
    if world == 1:
        return local
    out = torch.empty(world * local.numel(), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local, group=group)
    return out
