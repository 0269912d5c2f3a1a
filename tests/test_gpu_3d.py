"""GPU parity of the 3-D C-K-S operators (P:27,
P:407; reading c17) against the 3-D fp64 oracle (oracle/cks_oracle3d.py,
pinned in tests/test_oracle3d.py): ConvV2 with trimmed windows on the depth,
row and column axes, Stage1-free KS-deconv with sd*sh*sw phases, Sk-dilated
with leaping access on all three axes."""
import numpy as np
import pytest

from oracle import cks_oracle3d as O3
from oracle.cks_oracle import GeometryError, out_extent

from test_gpu_parity import TOL, U32, check, dev, torch_cuda  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


def _inputs(seed, N, C, OC, dhw, f, s, p, dtype):
    """Seeded U[-1,1) X / dY, kaiming-uniform W (the recipe of cks_synth),
    bf16-rounded for bf16."""
    import torch
    rng = np.random.default_rng(seed)
    O_ = [out_extent(i, ff, ss, pp) for i, ff, ss, pp in zip(dhw, f, s, p)]
    X = rng.uniform(-1, 1, (N, *dhw, C)).astype(np.float32)
    bound = 1.0 / np.sqrt(f[0] * f[1] * f[2] * C)
    W = rng.uniform(-bound, bound, (OC, *f, C)).astype(np.float32)
    G = rng.uniform(-1, 1, (N, *O_, OC)).astype(np.float32)
    if dtype == "bf16":
        X, W, G = (torch.from_numpy(a).bfloat16().float().numpy() for a in (X, W, G))
    return X, W, G


def _run3(torch, case, dtype, ops=("fwd", "deconv", "wgrad"), seed=0):
    from paper_2306_15951_b200 import ops as K
    N, C, OC, dhw, f, s, p = case
    X, W, G = _inputs(seed, N, C, OC, dhw, f, s, p, dtype)
    Xd, Wd, Gd = dev(torch, X, dtype), dev(torch, W, dtype), dev(torch, G, dtype)
    out = {}
    if "fwd" in ops:
        out["fwd"] = K.conv3d_fwd(Xd, Wd, s, p)
    if "deconv" in ops:
        out["deconv"] = K.deconv3d(Gd, Wd, dhw, s, p)
    if "wgrad" in ops:
        out["wgrad"] = K.dilated_wgrad3d(Xd, Gd, f, s, p)
    torch.cuda.synchronize()
    got = {k: v.cpu().numpy() for k, v in out.items()}
    red = {"fwd": f[0] * f[1] * f[2] * C, "deconv": f[0] * f[1] * f[2] * OC,
           "wgrad": N * int(np.prod(G.shape[1:4]))}
    if "fwd" in got:
        check(got["fwd"], O3.conv3d_ref(X, W, s, p), dtype, f"{case} conv3d", red["fwd"])
    if "deconv" in got:
        check(got["deconv"], O3.deconv3d_ref(G, W, dhw, s, p), dtype, f"{case} deconv3d", red["deconv"])
    if "wgrad" in got:
        check(got["wgrad"], O3.wgrad3d_ref(X, G, f, s, p), dtype, f"{case} wgrad3d", red["wgrad"])
    return got


def _rand_cases(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        f = tuple(int(rng.choice([1, 2, 3, 4, 5])) for _ in range(3))
        s = tuple(int(rng.integers(1, 4)) for _ in range(3))
        p = tuple(int(rng.integers(0, ff)) for ff in f)
        dhw = tuple(int(rng.integers(2, 13)) for _ in range(3))
        try:
            [out_extent(i, ff, ss, pp) for i, ff, ss, pp in zip(dhw, f, s, p)]
        except GeometryError:
            continue
        C = int(rng.choice([8, 16, 24, 64, 72]))
        OC = int(rng.choice([5, 8, 32, 64, 96]))
        N = int(rng.choice([1, 3, 130]))
        if N * np.prod(dhw) * max(C, OC) > 2.5e6:
            continue
        out.append((N, C, OC, dhw, f, s, p))
    return out


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("k", range(14))
def test_3d_random(torch_cuda, dtype, k):
    case = _rand_cases(14, 61 if dtype == "bf16" else 67)[k]
    _run3(torch_cuda, case, dtype, seed=k)


CASES = {
    # R3D-style layers (3-D ResNet: 3x3x3, stride 1 / 2), clips of 8-16 frames
    "r3d_s1": (130, 64, 64, (8, 14, 14), (3, 3, 3), (1, 1, 1), (1, 1, 1)),
    "r3d_s2": (130, 64, 128, (8, 14, 14), (3, 3, 3), (2, 2, 2), (1, 1, 1)),
    "r3d_ds": (130, 64, 128, (8, 14, 14), (1, 1, 1), (2, 2, 2), (0, 0, 0)),
    # 3-D generator / U-Net up-sampling: 4x4x4 s2 p1 (the DCGAN shape in 3-D)
    "gen3d": (66, 64, 32, (8, 8, 8), (4, 4, 4), (2, 2, 2), (1, 1, 1)),
    # depth-only stride, (1, 3, 3) filters (factorised (2+1)-D style)
    "d_only": (40, 32, 48, (9, 10, 11), (3, 1, 1), (2, 1, 1), (1, 0, 0)),
    "hw_only": (40, 32, 48, (5, 10, 11), (1, 3, 3), (1, 2, 2), (0, 1, 1)),
    # stem-like narrow input channels (channel-padded staging for fwd / wgrad)
    "stem3d": (20, 3, 64, (8, 32, 32), (3, 7, 7), (1, 2, 2), (1, 3, 3)),
}


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("name", list(CASES))
def test_3d_layers(torch_cuda, name, dtype):
    case = CASES[name]
    ops = ("fwd", "wgrad") if case[1] * (2 if dtype == "bf16" else 4) % 16 else ("fwd", "deconv", "wgrad")
    _run3(torch_cuda, case, dtype, ops=ops, seed=7)


def test_3d_trivial_depth_equals_2d(torch_cuda):
    """D = F_D = 1: the 3-D entry points give the 2-D operators' results bit for bit
    (same plans up to the trivial depth table)."""
    torch = torch_cuda
    from paper_2306_15951_b200 import ops as K
    X, W, G = _inputs(3, 131, 64, 96, (1, 9, 10), (1, 3, 3), (1, 2, 2), (0, 1, 1), "bf16")
    Xd, Wd, Gd = dev(torch, X, "bf16"), dev(torch, W, "bf16"), dev(torch, G, "bf16")
    y3 = K.conv3d_fwd(Xd, Wd, (1, 2, 2), (0, 1, 1))[:, 0]
    y2 = K.conv2d_fwd(Xd[:, 0].contiguous(), Wd[:, 0].contiguous(), (2, 2), (1, 1))
    x3 = K.deconv3d(Gd, Wd, (1, 9, 10), (1, 2, 2), (0, 1, 1))[:, 0]
    x2 = K.deconv2d(Gd[:, 0].contiguous(), Wd[:, 0].contiguous(), (9, 10), (2, 2), (1, 1), ks_mode="stage1_free")
    w3 = K.dilated_wgrad3d(Xd, Gd, (1, 3, 3), (1, 2, 2), (0, 1, 1))[:, 0]
    w2 = K.dilated_wgrad(Xd[:, 0].contiguous(), Gd[:, 0].contiguous(), (3, 3), (2, 2), (1, 1))
    torch.cuda.synchronize()
    assert torch.equal(y3, y2) and torch.equal(x3, x2) and torch.equal(w3, w2)


def test_3d_deconv_unsupported_narrow_rows(torch_cuda):
    """KS-deconv 3-D reads W directly: W rows of 6 bytes (C = 3, bf16) are refused."""
    torch = torch_cuda
    from paper_2306_15951_b200 import _lib as L
    from paper_2306_15951_b200 import ops as K
    W = torch.zeros((8, 3, 3, 3, 3), dtype=torch.bfloat16, device="cuda")
    G = torch.zeros((2, 4, 4, 4, 8), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(L.CksError):
        K.deconv3d(G, W, (8, 8, 8), 2, 1)


RG_CASES = {
    # small clip batches (row groups of 4 / 2 h rows x 32 / 64 clips inside each depth slice)
    "rg_r3d_s1": (8, 64, 64, (8, 14, 14), (3, 3, 3), (1, 1, 1), (1, 1, 1)),
    "rg_r3d_s2": (24, 64, 128, (8, 15, 13), (3, 3, 3), (2, 2, 2), (1, 1, 1)),
    "rg_gen3d": (33, 64, 32, (6, 8, 8), (4, 4, 4), (2, 2, 2), (1, 1, 1)),
    "rg_hw_s3": (64, 32, 48, (5, 19, 11), (1, 3, 3), (1, 3, 2), (0, 1, 1)),
}


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("name", list(RG_CASES))
def test_3d_row_groups(torch_cuda, name, dtype):
    """3-D ConvV2 / KS-deconv at N <= 64: row groups of h rows inside each depth slice (the same
    grouping as the 2-D plane, whose plan reports rg = 32 / 64 for these batches)."""
    from paper_2306_15951_b200 import _lib as L
    case = RG_CASES[name]
    N, C, OC, dhw, f, s, p = case
    plane = L.make_geom(N, C, dhw[1], dhw[2], OC, f[1], f[2], s[1], s[2], p[1], p[2])
    assert int(L.plan_dict(plane, L.CKS_BF16, L.CKS_OP_FWD)["rg"]) == (32 if N <= 32 else 64)
    _run3(torch_cuda, case, dtype, ops=("fwd", "deconv"), seed=11)
