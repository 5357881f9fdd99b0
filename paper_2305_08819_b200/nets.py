"""Conv layer shapes of the paper's CIFAR-10 networks (pure data, no arithmetic).

The paper trains AlexNet, VGG-16/19, GoogLeNet and ResNet-18/34 on CIFAR-10
(Table III; inputs 32x32x3, batch 512) but never
lists their layers.  These per-layer tables are this build's CIFAR adaptations
(BASELINE.json configs 2-5), including the 3x3 stride-2
downsample of Fig. 2's Block(64,128,2).

A layer is (name, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw, ic_logical);
IC is already padded to a multiple of 4 ("padded to 4x"), the
logical count is kept for the Kaiming fan-in.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List


@dataclass(frozen=True)
class Layer:
    name: str
    IH: int
    IW: int
    IC: int
    OC: int
    FH: int
    FW: int
    sh: int
    sw: int
    ph: int
    pw: int
    ic_logical: int

    @property
    def OH(self) -> int:
        return (self.IH + 2 * self.ph - self.FH) // self.sh + 1

    @property
    def OW(self) -> int:
        return (self.IW + 2 * self.pw - self.FW) // self.sw + 1

    def dims(self, N: int):
        """The C-ABI argument tuple (N,IH,IW,IC,OC,FH,FW,sh,sw,ph,pw)."""
        return (N, self.IH, self.IW, self.IC, self.OC, self.FH, self.FW,
                self.sh, self.sw, self.ph, self.pw)


def _pad4(c: int) -> int:
    return (c + 3) // 4 * 4


def L(name, H, IC, OC, k=3, s=1, p=None, W=None):
    if p is None:
        p = k // 2
    return Layer(name, H, H if W is None else W, _pad4(IC), OC, k, k, s, s, p, p, IC)


def vgg16() -> List[Layer]:
    """VGG-16 CIFAR: cfg 64,64,M,128,128,M,256x3,M,512x3,M,512x3,M; all 3x3 s1 p1."""
    return [
        L("vgg1", 32, 3, 64), L("vgg2", 32, 64, 64),
        L("vgg3", 16, 64, 128), L("vgg4", 16, 128, 128),
        L("vgg5", 8, 128, 256), L("vgg6", 8, 256, 256), L("vgg7", 8, 256, 256),
        L("vgg8", 4, 256, 512), L("vgg9", 4, 512, 512), L("vgg10", 4, 512, 512),
        L("vgg11", 2, 512, 512), L("vgg12", 2, 512, 512), L("vgg13", 2, 512, 512),
    ]


def resnet18(hw: int = 32) -> List[Layer]:
    """ResNet-18 CIFAR (3x3 stem at 32x32, 4 stages of 2 BasicBlocks), in forward order.

    Each stage change has a 3x3 stride-2 conv and a 1x1 stride-2 p0 shortcut.
    20 convs: 17 3x3 + 3 1x1.  `hw` != 32: the same network on larger inputs -- the large-map regime
    where the paper reports cu32 losing to cuDNN ("when the input-feature-size >= 128 x 128",
    PAPER.md:169).
    """
    out = [L("conv1", hw, 3, 64)]
    H, C = hw, 64
    for stage, OC in ((1, 64), (2, 128), (3, 256), (4, 512)):
        for blk in range(2):
            if blk == 0 and stage > 1:
                out.append(L("l%d.%da" % (stage, blk), H, C, OC, s=2))
                out.append(L("l%d.%dsc" % (stage, blk), H, C, OC, k=1, s=2, p=0))
                H //= 2
            else:
                out.append(L("l%d.%da" % (stage, blk), H, C, OC))
            out.append(L("l%d.%db" % (stage, blk), H, OC, OC))
            C = OC
    return out


def alexnet() -> List[Layer]:
    """AlexNet-CIFAR: 11x11 s4 p5, 5x5 p2 at 4x4, 3x3 at 2x2."""
    return [
        Layer("alex1", 32, 32, 4, 64, 11, 11, 4, 4, 5, 5, 3),
        L("alex2", 4, 64, 192, k=5),
        L("alex3", 2, 192, 384), L("alex4", 2, 384, 256), L("alex5", 2, 256, 256),
    ]


_INCEPTION = [  # name, H, in, b1, b2r, b2, b3r, b3, b4
    ("a3", 32, 192, 64, 96, 128, 16, 32, 32),
    ("b3", 32, 256, 128, 128, 192, 32, 96, 64),
    ("a4", 16, 480, 192, 96, 208, 16, 48, 64),
    ("b4", 16, 512, 160, 112, 224, 24, 64, 64),
    ("c4", 16, 512, 128, 128, 256, 24, 64, 64),
    ("d4", 16, 512, 112, 144, 288, 32, 64, 64),
    ("e4", 16, 528, 256, 160, 320, 32, 128, 128),
    ("a5", 8, 832, 256, 160, 320, 32, 128, 128),
    ("b5", 8, 832, 384, 192, 384, 48, 128, 128),
]


def googlenet() -> List[Layer]:
    """GoogLeNet-CIFAR: 3x3 stem 3->192, inception a3..b5 (original table), real 5x5 p2. 55 convs."""
    out = [L("g.stem", 32, 3, 192)]
    for name, H, cin, b1, b2r, b2, b3r, b3, b4 in _INCEPTION:
        out += [L("g.%s.1x1" % name, H, cin, b1, k=1),
                L("g.%s.3x3r" % name, H, cin, b2r, k=1), L("g.%s.3x3" % name, H, b2r, b2),
                L("g.%s.5x5r" % name, H, cin, b3r, k=1), L("g.%s.5x5" % name, H, b3r, b3, k=5),
                L("g.%s.pool" % name, H, cin, b4, k=1)]
    return out


NETS = {"vgg16": vgg16, "resnet18": resnet18, "alexnet": alexnet, "googlenet": googlenet,
        # large-map regime: the CIFAR ResNet-18 on 64 / 128 / 224-pixel inputs
        "resnet18@64": lambda: resnet18(64), "resnet18@128": lambda: resnet18(128),
        "resnet18@224": lambda: resnet18(224)}


def valid_pairs(layer: Layer) -> int:
    """Number of in-bounds (output position, tap) pairs per image."""
    def count(I, O, F, s, p):
        return sum(1 for o in range(O) for f in range(F) if 0 <= o * s - p + f < I)
    return (count(layer.IH, layer.OH, layer.FH, layer.sh, layer.ph) *
            count(layer.IW, layer.OW, layer.FW, layer.sw, layer.pw))


def flops(layer: Layer, N: int, valid: bool = True) -> int:
    """Algorithmic FLOPs of one op (fwd, dX or dW — identical pair sets): 2 * pairs * IC * OC.

    Uses the LOGICAL input channels (pad lanes are not work)."""
    pairs = valid_pairs(layer) if valid else layer.OH * layer.OW * layer.FH * layer.FW
    return 2 * N * pairs * layer.ic_logical * layer.OC


def touched_rows(I: int, O: int, F: int, s: int, p: int) -> int:
    """Input rows (or columns) some (output, tap) pair reads: a 1x1 stride-2 conv touches every
    other row, a 3x3 stride-2 pad-1 conv all of them."""
    return sum(1 for i in range(I) if any(0 <= (i + p - f) and (i + p - f) % s == 0 and (i + p - f) // s < O
                                          for f in range(F)))


def bytes_compulsory(layer: Layer, N: int, op: str) -> int:
    """Compulsory fp32 bytes: fwd X(touched) + W + Y; dX dY + W + dX (all of dX is
    written, zeros included); dW X(touched) + dY + dW.  Each input read once, each output written once."""
    x_all = N * layer.IH * layer.IW * layer.IC * 4
    x = (N * touched_rows(layer.IH, layer.OH, layer.FH, layer.sh, layer.ph)
         * touched_rows(layer.IW, layer.OW, layer.FW, layer.sw, layer.pw) * layer.IC * 4)
    y = N * layer.OH * layer.OW * layer.OC * 4
    w = layer.OC * layer.FH * layer.FW * layer.IC * 4
    if op == "fwd":
        return x + w + y
    if op == "dx":
        return y + w + x_all
    if op == "dw":
        return x + y + w
    raise ValueError(op)
