"""Multi-GPU sharding of the HE convolution by output channel.

One process per GPU. Every rank holds the same input ciphertexts (the client's upload is
broadcast once) and the same layer plan (computed for the FULL output-channel count M, so the
packing of the inputs does not depend on the number of ranks); rank k owns the contiguous
output-channel slice [m0, m0 + mc) of every layer: it preprocesses only those weights, runs
secn_he_conv2d on a plan copy with M = mc, and extracts its part of the server's output share.
The only collective is an all-gather of those shares (the north star's "NCCL all-gather over
NVLink only to collect output shares"); output ciphertexts stay on the rank that computed them.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Tuple

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


def padded_slice(M: int, world: int) -> int:
    """Rows per rank in the all-gather buffer (all-gather needs equal sizes)."""
    return -(-M // world)


@dataclass
class ShareLayout:
    """Where each layer's share block lives in one flat per-step all-gather buffer."""
    offsets: List[int]       # per layer, offset (elements) within a rank's chunk
    sizes: List[int]         # per layer, padded rows * OH * OW
    chunk: int               # elements per rank


def share_layout(dims: List[Tuple[int, int, int]], world: int) -> ShareLayout:
    """dims = [(M, OH, OW)] per layer."""
    offs, sizes, o = [], [], 0
    for M, OH, OW in dims:
        sz = padded_slice(M, world) * OH * OW
        offs.append(o)
        sizes.append(sz)
        o += sz
    return ShareLayout(offs, sizes, o)


def reassemble(gathered: torch.Tensor, layout: ShareLayout, dims: List[Tuple[int, int, int]], world: int
               ) -> List[torch.Tensor]:
    """gathered [world * chunk] -> per layer full share tensor [M, OH, OW] (drops padding)."""
    g = gathered.view(world, layout.chunk)
    out = []
    for (M, OH, OW), off, sz in zip(dims, layout.offsets, layout.sizes):
        rows = padded_slice(M, world)
        blocks = []
        for k, (m0, mc) in enumerate(m_slices(M, world)):
            blocks.append(g[k, off:off + sz].view(rows, OH, OW)[:mc])
        out.append(torch.cat(blocks, 0))
    return out


def all_gather_shares(local: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """local [chunk] -> [world * chunk] via one all_gather_into_tensor (NCCL on GPUs)."""
    if world == 1:
        return local
    out = torch.empty(world * local.numel(), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local, group=group)
    return out
