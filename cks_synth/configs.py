"""Workload shapes (BASELINE.json ``configs``).

Only shapes live here -- no arithmetic of the method.  ``Layer`` uses the
paper's Table I notation: N, I_C(=C), I_H(=H), I_W(=W), O_C,
F_H, F_W, sh, sw, ph, pw.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

ALL_OPS = ("fwd", "deconv", "wgrad")


@dataclass(frozen=True)
class Layer:
    name: str
    N: int
    C: int
    H: int
    W: int
    OC: int
    FH: int
    FW: int
    sh: int
    sw: int
    ph: int
    pw: int
    ops: tuple = ALL_OPS

    def out_hw(self):
        # Table I output extent (floor rounding, SURVEY.md §8(c) reading c10).
        return ((self.H + 2 * self.ph - self.FH) // self.sh + 1,
                (self.W + 2 * self.pw - self.FW) // self.sw + 1)

    def with_batch(self, n: int) -> "Layer":
        return replace(self, N=n)

    def geom(self):
        return dict(N=self.N, C=self.C, H=self.H, W=self.W, OC=self.OC, FH=self.FH,
                    FW=self.FW, sh=self.sh, sw=self.sw, ph=self.ph, pw=self.pw)


def _c1():
    return [Layer("c1_tiny", 2, 4, 8, 8, 8, 3, 3, 2, 2, 1, 1)]


def _c2(N=128):
    shapes = [(32, 3, 64), (32, 64, 64), (16, 64, 128), (16, 128, 128),
              (8, 128, 256), (8, 256, 256), (4, 256, 512), (4, 512, 512)]
    out = []
    for (I, ic, oc) in shapes:
        for s in (1, 2):
            out.append(Layer(f"vgg{I}_{ic}to{oc}_s{s}", N, ic, I, I, oc, 3, 3, s, s, 1, 1))
    return out


def _c3(N=256):
    L = []
    L.append(Layer("stem", N, 3, 224, 224, 64, 7, 7, 2, 2, 3, 3, ("fwd", "wgrad")))
    for i in range(4):
        L.append(Layer(f"l1_{i}", N, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1))
    L.append(Layer("l2a", N, 64, 56, 56, 128, 3, 3, 2, 2, 1, 1))
    L.append(Layer("l2ds", N, 64, 56, 56, 128, 1, 1, 2, 2, 0, 0))
    for i in range(3):
        L.append(Layer(f"l2_{i}", N, 128, 28, 28, 128, 3, 3, 1, 1, 1, 1))
    L.append(Layer("l3a", N, 128, 28, 28, 256, 3, 3, 2, 2, 1, 1))
    L.append(Layer("l3ds", N, 128, 28, 28, 256, 1, 1, 2, 2, 0, 0))
    for i in range(3):
        L.append(Layer(f"l3_{i}", N, 256, 14, 14, 256, 3, 3, 1, 1, 1, 1))
    L.append(Layer("l4a", N, 256, 14, 14, 512, 3, 3, 2, 2, 1, 1))
    L.append(Layer("l4ds", N, 256, 14, 14, 512, 1, 1, 2, 2, 0, 0))
    for i in range(3):
        L.append(Layer(f"l4_{i}", N, 512, 7, 7, 512, 3, 3, 1, 1, 1, 1))
    return L


def _c4(N=512):
    # Conv-layer view: X = the generator's big side; KS-deconv is the
    # generator forward (dY := z), Sk-dilated its weight gradient.
    ops = ("deconv", "wgrad")
    return [Layer("G4to8", N, 512, 8, 8, 1024, 4, 4, 2, 2, 1, 1, ops),
            Layer("G8to16", N, 256, 16, 16, 512, 4, 4, 2, 2, 1, 1, ops),
            Layer("G16to32", N, 128, 32, 32, 256, 4, 4, 2, 2, 1, 1, ops),
            Layer("G32to64", N, 3, 64, 64, 128, 4, 4, 2, 2, 1, 1, ops)]


def _c6(N=128):
    # The paper's second operator test set (Exp. 1, Figs 10/12/14):
    # 5x5 filters, padding 2, 8 cases with shrinking maps and growing channels.
    # The per-case shapes are not printed (figures missing), so this follows
    # the C2 progression, strides 1 and 2.
    shapes = [(32, 64, 64), (16, 64, 128), (16, 128, 128), (8, 128, 256),
              (8, 256, 256), (4, 256, 512), (4, 512, 512), (32, 3, 64)]
    out = []
    for (I, ic, oc) in shapes:
        for s in (1, 2):
            out.append(Layer(f"f5_{I}_{ic}to{oc}_s{s}", N, ic, I, I, oc, 5, 5, s, s, 2, 2))
    return out


CONFIGS = {
    0: ("C1 tiny: N=2 C=4 8x8 OC=8 3x3 s2 p1", _c1),
    1: ("C2 Cifar10 VGG-16 layer sweep N=128, 3x3 p1, s1/s2", _c2),
    2: ("C3 ILSVRC2012 ResNet-18 conv layers N=256 @224", _c3),
    3: ("C4 DCGAN generator 4x4 s2 p1 N=512 (KS-deconv + Sk-dilated)", _c4),
    # C5 (configs[4]) is the C3 layer list as a full train step, batch-sharded.
    4: ("C5 ResNet-18 conv-layer train step, batch-sharded, NCCL wgrad allreduce", _c3),
    5: ("C6 5x5 p2 layer sweep (the paper's second test set) N=128, s1/s2", _c6),
}


def get_config(idx: int, N: int | None = None):
    desc, fn = CONFIGS[idx]
    layers = fn() if N is None or idx == 0 else fn(N)
    return desc, layers
