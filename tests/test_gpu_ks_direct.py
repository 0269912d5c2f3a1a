"""GPU parity of the Stage1-free KS-deconv (the
all-in-one variant the paper set aside): the implicit GEMM reads W
itself as an MN-major B operand, the taps of sub-filter row ch of phase (y, x)
being fw = x, x+sw, ... of filter row fh = y + (CH_y-1-ch)*sh (Alg. 2 Stage1's
index map, Fig. 5) -- no packed sub-filters.  Forced through
cks_deconv2d_ex(CKS_KS_STAGE1_FREE) and compared with the fp64 oracle's
zero-inserting definition (Eq 2) and with the Stage1 path."""
import numpy as np
import pytest

import oracle as O
from cks_synth import Layer, get_config, make_layer_inputs

from test_gpu_parity import check, dev, red_len, torch_cuda  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


def _deconv(torch, lay, dtype, config, idx, mode):
    from paper_2306_15951_b200 import ops as K
    a = make_layer_inputs(lay, config, idx, dtype)
    G, W = dev(torch, a["dY"], dtype), dev(torch, a["W"], dtype)
    dx = K.deconv2d(G, W, (lay.H, lay.W), (lay.sh, lay.sw), (lay.ph, lay.pw), ks_mode=mode)
    torch.cuda.synchronize()
    return a, dx.cpu().numpy()


def _layers(n, seed, dtype):
    rng = np.random.default_rng(seed)
    out = []
    q = 8 if dtype == "bf16" else 4
    while len(out) < n:
        FH, FW = int(rng.choice([1, 2, 3, 4, 5, 7])), int(rng.choice([1, 2, 3, 4, 5, 7]))
        sh, sw = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        ph, pw = int(rng.integers(0, FH)), int(rng.integers(0, FW))
        H, W = int(rng.integers(max(1, FH - 2 * ph), 22)), int(rng.integers(max(1, FW - 2 * pw), 22))
        C = int(rng.choice([q, 2 * q, 24, 64, 72, 136]))          # W rows: 16-byte multiples
        OC = int(rng.choice([3, 5, 8, 32, 64, 96, 200]))
        N = int(rng.choice([1, 5, 130]))
        lay = Layer(f"kd{len(out)}", N, C, H, W, OC, FH, FW, sh, sw, ph, pw)
        try:
            O.geom(**lay.geom())
        except O.GeometryError:
            continue
        if N * H * W * max(C, OC) > 3e6:
            continue
        out.append(lay)
    return out


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("k", range(16))
def test_stage1_free_random(torch_cuda, dtype, k):
    lay = _layers(16, 41 if dtype == "bf16" else 43, dtype)[k]
    a, got = _deconv(torch_cuda, lay, dtype, 24, k, "stage1_free")
    ref = O.deconv_ref(a["dY"], a["W"], lay.H, lay.W, lay.sh, lay.sw, lay.ph, lay.pw)
    check(got, ref, dtype, f"{lay} stage1-free deconv", red_len(lay, "deconv"))


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("lay", [Layer("e_ds", 131, 64, 8, 8, 128, 1, 1, 2, 2, 0, 0),    # empty phase (c11)
                                 Layer("e_tail", 3, 16, 6, 7, 24, 3, 3, 2, 2, 0, 0),    # unread rows (c10)
                                 Layer("e_s3", 67, 32, 13, 11, 40, 5, 4, 3, 3, 2, 1),   # CW_x differs per phase
                                 Layer("e_dc", 130, 64, 16, 16, 128, 4, 4, 2, 2, 1, 1),  # DCGAN (negative oh_s)
                                 Layer("e_f7", 70, 8, 20, 20, 16, 7, 7, 4, 4, 3, 3),    # s > F/2, narrow IC
                                 Layer("e_wide", 130, 192, 9, 9, 72, 3, 3, 2, 2, 1, 1),  # several N atoms per tap
                                 Layer("e_w5", 129, 256, 8, 8, 136, 5, 5, 2, 2, 2, 2)],  # (5-D W map), OC ragged
                         ids=lambda l: l.name)
def test_stage1_free_edges(torch_cuda, lay, dtype):
    a, got = _deconv(torch_cuda, lay, dtype, 25, 0, "stage1_free")
    ref = O.deconv_ref(a["dY"], a["W"], lay.H, lay.W, lay.sh, lay.sw, lay.ph, lay.pw)
    check(got, ref, dtype, f"{lay.name} stage1-free deconv", red_len(lay, "deconv"))
    if lay.name == "e_ds":
        assert np.all(got[:, 1::2, :, :] == 0) and np.all(got[:, :, 1::2, :] == 0)
    _, s1 = _deconv(torch_cuda, lay, dtype, 25, 0, "stage1")
    check(got, s1, dtype, f"{lay.name} stage1-free vs stage1", red_len(lay, "deconv"))


def _config_deconv_layers():
    out = []
    for cfg in (1, 2, 3):
        for i, lay in enumerate(get_config(cfg)[1]):
            if "deconv" not in lay.ops or lay.C * 2 % 16:
                continue
            if lay.name.startswith(("l1_", "l2_", "l3_", "l4_")) and not lay.name.endswith("_0"):
                continue
            out.append((cfg, i, lay))
    return out


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("cfg,i,lay", _config_deconv_layers(), ids=lambda v: v.name if isinstance(v, Layer) else str(v))
def test_stage1_free_config_layers(torch_cuda, cfg, i, lay, dtype):
    """Every config KS-deconv layer with 16-byte W rows, Stage1-free, reduced batch."""
    small = lay.with_batch(130 if lay.H * lay.W * max(lay.C, lay.OC) < 2e5 else 3)
    a, got = _deconv(torch_cuda, small, dtype, cfg, i, "stage1_free")
    ref = O.deconv_ref(a["dY"], a["W"], small.H, small.W, small.sh, small.sw, small.ph, small.pw)
    check(got, ref, dtype, f"{lay.name} stage1-free deconv", red_len(small, "deconv"))
