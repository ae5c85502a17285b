"""Layer scheduling for a network's HE-linear layers on one GPU: which layers the network's
data flow lets the server run at the same time, and a stream fork/join executor for them.

The server evaluates a network's convolutions one layer at a time because each layer's input
share comes out of the nonlinear protocol that follows the previous one (§7).
Two layers that read the SAME input tensor are independent:
  * SqueezeNet fire modules: expand1x1 (``fireK.e1``) and expand3x3 (``fireK.e3``) both read the
    squeeze output (their results are concatenated afterwards);
  * ResNet bottleneck blocks with a projection: ``lX.b0.c1`` and ``lX.b0.ds`` both read the
    block input.
Only such groups overlap (on separate CUDA streams); everything else keeps the network order,
so the step time stays what the protocol would see layer by layer.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence

import torch


def concurrent_groups(names: Sequence[str]) -> List[List[int]]:
    """Partitions layer indices into groups that may run concurrently, ordered by each group's
    first layer. A later member moves up to its group (valid: it reads the same input as the
    group's first layer, which is ready then), e.g. a ResNet projection ``ds`` runs beside ``c1``."""
    groups: List[List[int]] = []
    key_of = {}
    for i, n in enumerate(names):
        key = None
        if n.endswith(".e1") or n.endswith(".e3"):
            key = ("fire", n[:-3])
        elif n.endswith(".b0.c1") or n.endswith(".b0.ds"):
            key = ("proj", n.rsplit(".", 1)[0])
        if key is not None and key in key_of:  # same input as an earlier layer: joins its group
            groups[key_of[key]].append(i)
            continue
        if key is not None:
            key_of[key] = len(groups)
        groups.append([i])
    return groups


class GroupRunner:
    """Runs ``fn(i)`` for every layer index in ``groups``: a group's first layer on the current
    stream, the others on side streams forked from it and joined back before the next group.
    Works eagerly and under CUDA-graph capture (the fork/join become graph edges)."""

    def __init__(self, groups: List[List[int]], device, priority: int = 0):
        self.groups = groups
        width = max((len(g) for g in groups), default=1)
        self.side = [torch.cuda.Stream(device, priority=priority) for _ in range(width - 1)]

    def __call__(self, fn: Callable[[int], None], before_group: Optional[Callable[[int], None]] = None) -> None:
        """before_group(k), if given, runs on the host before group k is issued (e.g. to issue side
        work the group's layers wait for)."""
        for k, g in enumerate(self.groups):
            if before_group is not None:
                before_group(k)
            self.run_group(g, fn)

    def run_group(self, g: List[int], fn: Callable[[int], None]) -> None:
        main = torch.cuda.current_stream()
        if len(g) == 1:
            fn(g[0])
            return
        for s in self.side[:len(g) - 1]:
            s.wait_stream(main)
        for s, i in zip(self.side, g[1:]):
            with torch.cuda.stream(s):
                fn(i)
        fn(g[0])
        for s in self.side[:len(g) - 1]:
            main.wait_stream(s)


class StagedGroupRunner:
    """Like GroupRunner, but a group's layers advance stage by stage: ``stage_fn(i, k)`` runs launch
    group k (0: share add + NTT, 1: MAC, 2: INTT tail + mask) of layer i, the group's layers run
    stage k concurrently on their streams, and the streams join before stage k + 1. So kernels of
    the same kind overlap (two MACs, two tails), but a tail never runs beside another layer's MAC --
    the overlap that produced wrong words in tools/race_check.py."""

    def __init__(self, groups: List[List[int]], device, n_stages: int = 3):
        self.groups = groups
        self.n_stages = n_stages
        width = max((len(g) for g in groups), default=1)
        self.side = [torch.cuda.Stream(device) for _ in range(width - 1)]

    def __call__(self, fn: Callable[[int], None], stage_fn: Optional[Callable[[int, int], None]] = None) -> None:
        """Without ``stage_fn`` (an entry point with no staged form) every layer runs whole, in order."""
        main = torch.cuda.current_stream()
        for g in self.groups:
            if len(g) == 1 or stage_fn is None:
                for i in g:
                    fn(i)
                continue
            for k in range(self.n_stages):
                for s in self.side[:len(g) - 1]:
                    s.wait_stream(main)
                for s, i in zip(self.side, g[1:]):
                    with torch.cuda.stream(s):
                        stage_fn(i, k)
                stage_fn(g[0], k)
                for s in self.side[:len(g) - 1]:
                    main.wait_stream(s)
