"""Convolution-layer geometry of the paper's workloads (shapes only; no HE arithmetic).

The paper evaluates all convolutions of a 37-bit quantised SqueezeNet on ImageNet
(§8; Table 5 at PAPER.md:461-482) and a ResNet50 (App. C.2).
It does not say which SqueezeNet version; reading R13 takes torchvision
SqueezeNet 1.1 as primary and 1.0 as secondary, both at 224x224.

Each layer is a ``ConvLayer(name, C, H, W, M, k, stride, pad)`` with a square k x k kernel,
input C x H x W and M output channels. This module is shared by the oracle side and the
CUDA side only as a table of shapes.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List


@dataclass(frozen=True)
class ConvLayer:
    name: str
    C: int
    H: int
    W: int
    M: int
    k: int
    stride: int = 1
    pad: int = 0

    @property
    def OH(self) -> int:
        return (self.H + 2 * self.pad - self.k) // self.stride + 1

    @property
    def OW(self) -> int:
        return (self.W + 2 * self.pad - self.k) // self.stride + 1


def _fire(name: str, C: int, HW: int, sq: int, e1: int, e3: int) -> List[ConvLayer]:
    return [
        ConvLayer(f"{name}.sq", C, HW, HW, sq, 1),
        ConvLayer(f"{name}.e1", sq, HW, HW, e1, 1),
        ConvLayer(f"{name}.e3", sq, HW, HW, e3, 3, 1, 1),
    ]


def squeezenet11() -> List[ConvLayer]:
    """torchvision SqueezeNet 1.1 conv layers at 224x224 (26 layers)."""
    L = [ConvLayer("conv1", 3, 224, 224, 64, 3, 2, 0)]  # -> 111, maxpool -> 55
    L += _fire("fire2", 64, 55, 16, 64, 64)
    L += _fire("fire3", 128, 55, 16, 64, 64)  # maxpool -> 27
    L += _fire("fire4", 128, 27, 32, 128, 128)
    L += _fire("fire5", 256, 27, 32, 128, 128)  # maxpool -> 13
    L += _fire("fire6", 256, 13, 48, 192, 192)
    L += _fire("fire7", 384, 13, 48, 192, 192)
    L += _fire("fire8", 384, 13, 64, 256, 256)
    L += _fire("fire9", 512, 13, 64, 256, 256)
    L.append(ConvLayer("conv10", 512, 13, 13, 1000, 1))
    return L


def squeezenet10() -> List[ConvLayer]:
    """torchvision SqueezeNet 1.0 conv layers at 224x224 (26 layers)."""
    L = [ConvLayer("conv1", 3, 224, 224, 96, 7, 2, 0)]  # -> 109, maxpool -> 54
    L += _fire("fire2", 96, 54, 16, 64, 64)
    L += _fire("fire3", 128, 54, 16, 64, 64)
    L += _fire("fire4", 128, 54, 32, 128, 128)  # maxpool -> 27
    L += _fire("fire5", 256, 27, 32, 128, 128)
    L += _fire("fire6", 256, 27, 48, 192, 192)
    L += _fire("fire7", 384, 27, 48, 192, 192)
    L += _fire("fire8", 384, 27, 64, 256, 256)  # maxpool -> 13
    L += _fire("fire9", 512, 13, 64, 256, 256)
    L.append(ConvLayer("conv10", 512, 13, 13, 1000, 1))
    return L


def resnet50() -> List[ConvLayer]:
    """torchvision ResNet-50 v1.5 conv layers at 224x224 (53 layers; stride on the 3x3)."""
    L = [ConvLayer("conv1", 3, 224, 224, 64, 7, 2, 3)]  # -> 112, maxpool -> 56
    cin, hw = 64, 56
    for li, (width, blocks, stride) in enumerate([(64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)], start=1):
        cout = 4 * width
        for b in range(blocks):
            s = stride if b == 0 else 1
            p = f"l{li}.b{b}"
            L.append(ConvLayer(f"{p}.c1", cin, hw, hw, width, 1))
            L.append(ConvLayer(f"{p}.c2", width, hw, hw, width, 3, s, 1))
            ohw = (hw + 2 - 3) // s + 1
            L.append(ConvLayer(f"{p}.c3", width, ohw, ohw, cout, 1))
            if b == 0:
                L.append(ConvLayer(f"{p}.ds", cin, hw, hw, cout, 1, s, 0))
            cin, hw = cout, ohw
    return L


def tiny() -> List[ConvLayer]:
    """BASELINE.json configs[0]: single 3x3 conv, 16x16x4 input -> 8 channels (pad 1)."""
    return [ConvLayer("tiny", 4, 16, 16, 8, 3, 1, 1)]


NETWORKS = {
    "tiny": tiny,
    "squeezenet1_1": squeezenet11,
    "squeezenet1_0": squeezenet10,
    "resnet50": resnet50,
}


def network(name: str) -> List[ConvLayer]:
    return NETWORKS[name]()
