"""Pins for the 3-D oracle (oracle/cks_oracle3d.py) against things other than
itself: torch's fp64 CPU conv3d / grad.conv3d_input / grad.conv3d_weight (the
textbook special case), scalar brute force, the adjoint identity, the
reduction to the pinned 2-D oracle when the depth axis is trivial, and the
zero-free MAC count against a brute-force enumeration of the non-zero terms.
CPU only."""
import numpy as np
import pytest

import oracle as O
from oracle import cks_oracle3d as O3


def _case(rng, max_i=7):
    while True:
        f = tuple(int(rng.choice([1, 2, 3, 4, 5])) for _ in range(3))
        s = tuple(int(rng.integers(1, 4)) for _ in range(3))
        p = tuple(int(rng.integers(0, ff)) for ff in f)
        dhw = tuple(int(rng.integers(1, max_i + 1)) for _ in range(3))
        try:
            [O.out_extent(i, ff, ss, pp) for i, ff, ss, pp in zip(dhw, f, s, p)]
        except O.GeometryError:
            continue
        return dict(N=int(rng.integers(1, 3)), C=int(rng.integers(1, 4)), OC=int(rng.integers(1, 4)), dhw=dhw,
                    f=f, s=s, p=p)


def _tensors(rng, c):
    O_ = [O.out_extent(i, ff, ss, pp) for i, ff, ss, pp in zip(c["dhw"], c["f"], c["s"], c["p"])]
    X = rng.uniform(-1, 1, (c["N"], *c["dhw"], c["C"]))
    W = rng.uniform(-1, 1, (c["OC"], *c["f"], c["C"]))
    G = rng.uniform(-1, 1, (c["N"], *O_, c["OC"]))
    return X, W, G


def test_against_torch_fp64():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(3)
    for _ in range(40):
        c = _case(rng, max_i=9)
        X, W, G = _tensors(rng, c)
        xt = torch.from_numpy(X).permute(0, 4, 1, 2, 3)
        wt = torch.from_numpy(W).permute(0, 4, 1, 2, 3)
        gt = torch.from_numpy(G).permute(0, 4, 1, 2, 3)
        y = torch.nn.functional.conv3d(xt, wt, stride=c["s"], padding=c["p"]).permute(0, 2, 3, 4, 1).numpy()
        np.testing.assert_allclose(O3.conv3d_ref(X, W, c["s"], c["p"]), y, rtol=0, atol=1e-12)
        dx = torch.nn.grad.conv3d_input(xt.shape, wt, gt, stride=c["s"], padding=c["p"]).permute(0, 2, 3, 4, 1)
        np.testing.assert_allclose(O3.deconv3d_ref(G, W, c["dhw"], c["s"], c["p"]), dx.numpy(), rtol=0, atol=1e-12)
        dw = torch.nn.grad.conv3d_weight(xt, wt.shape, gt, stride=c["s"], padding=c["p"]).permute(0, 2, 3, 4, 1)
        np.testing.assert_allclose(O3.wgrad3d_ref(X, G, c["f"], c["s"], c["p"]), dw.numpy(), rtol=0, atol=1e-12)


def test_brute_force_tiny():
    rng = np.random.default_rng(4)
    for _ in range(12):
        c = _case(rng, max_i=5)
        X, W, G = _tensors(rng, c)
        np.testing.assert_allclose(O3.conv3d_ref(X, W, c["s"], c["p"]), O3.brute_conv3d(X, W, c["s"], c["p"]),
                                   rtol=0, atol=1e-12)
        np.testing.assert_allclose(O3.deconv3d_ref(G, W, c["dhw"], c["s"], c["p"]),
                                   O3.brute_deconv3d(G, W, c["dhw"], c["s"], c["p"]), rtol=0, atol=1e-12)
        np.testing.assert_allclose(O3.wgrad3d_ref(X, G, c["f"], c["s"], c["p"]),
                                   O3.brute_wgrad3d(X, G, c["f"], c["s"], c["p"]), rtol=0, atol=1e-12)


def test_adjoint_identity():
    """<conv(X,W),G> = <X,deconv(G,W)> = <W,wgrad(X,G)> (chain rule)."""
    rng = np.random.default_rng(5)
    for _ in range(30):
        c = _case(rng)
        X, W, G = _tensors(rng, c)
        a = np.sum(O3.conv3d_ref(X, W, c["s"], c["p"]) * G)
        b = np.sum(X * O3.deconv3d_ref(G, W, c["dhw"], c["s"], c["p"]))
        d = np.sum(W * O3.wgrad3d_ref(X, G, c["f"], c["s"], c["p"]))
        assert abs(a - b) <= 1e-10 * max(1, abs(a)) and abs(a - d) <= 1e-10 * max(1, abs(a))


def test_trivial_depth_reduces_to_2d():
    """D = F_D = 1 (s_d = 1, p_d = 0): the 3-D definitions are the pinned 2-D ones."""
    rng = np.random.default_rng(6)
    for _ in range(20):
        c = _case(rng)
        c["dhw"], c["f"], c["s"], c["p"] = (1,) + c["dhw"][1:], (1,) + c["f"][1:], (1,) + c["s"][1:], (0,) + c["p"][1:]
        X, W, G = _tensors(rng, c)
        s2 = (c["s"][1], c["s"][2], c["p"][1], c["p"][2])
        np.testing.assert_allclose(O3.conv3d_ref(X, W, c["s"], c["p"])[:, 0], O.conv_ref(X[:, 0], W[:, 0], *s2),
                                   rtol=0, atol=1e-12)
        np.testing.assert_allclose(O3.deconv3d_ref(G, W, c["dhw"], c["s"], c["p"])[:, 0],
                                   O.deconv_ref(G[:, 0], W[:, 0], c["dhw"][1], c["dhw"][2], *s2), rtol=0, atol=1e-12)
        np.testing.assert_allclose(O3.wgrad3d_ref(X, G, c["f"], c["s"], c["p"])[:, 0],
                                   O.wgrad_ref(X[:, 0], G[:, 0], c["f"][1], c["f"][2], *s2), rtol=0, atol=1e-12)


def test_zero_free_count_by_enumeration():
    """N*C*OC*V_D*V_H*V_W equals the number of non-zero-operand products of
    the 3-D definition (brute-force enumeration of (o, f) triples)."""
    rng = np.random.default_rng(7)
    for _ in range(25):
        c = _case(rng)
        cnt = O3.op_counts3d(c["N"], c["C"], c["OC"], c["dhw"], c["f"], c["s"], c["p"])
        O_ = cnt["O"]
        n = 0
        for od in range(O_[0]):
            for oh in range(O_[1]):
                for ow in range(O_[2]):
                    for fd in range(c["f"][0]):
                        for fh in range(c["f"][1]):
                            for fw in range(c["f"][2]):
                                i = (od * c["s"][0] + fd - c["p"][0], oh * c["s"][1] + fh - c["p"][1],
                                     ow * c["s"][2] + fw - c["p"][2])
                                n += all(0 <= ii < I for ii, I in zip(i, c["dhw"]))
        assert cnt["zero_free_macs"] == c["N"] * c["C"] * c["OC"] * n
        assert cnt["zero_free_macs"] <= min(cnt["nominal_macs_conv"], cnt["nominal_macs_deconv"],
                                            cnt["nominal_macs_dilated"])
