"""GPU parity over the paper's general operator space and a full DCGAN
generator step.

* The F in {1..7} x s in {1..4} grid (the strides and filter sizes the C-K-S
  formulas are stated for, Alg. 1-3B): all three
  operators, against the fp64 oracle, in BF16 and TF32.
* A whole DCGAN generator (the C4 widths, 4x4 s2 p1, "deconvolutional
  layers") trained through CKSConvTranspose2dFunction: forward = KS-deconv of
  every layer in sequence, backward = ConvV2 (input gradient) + Sk-dilated
  (weight gradient) of every layer; each layer checked against the oracle
  on the tensors the chain actually fed it.
"""
import numpy as np
import pytest

import oracle as O
from cks_synth import Layer, bf16_bits, make_layer_inputs

from test_gpu_parity import TOL, check, check_full, dev, red_len, torch_cuda  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


def _grid():
    out = []
    for F in range(1, 8):
        for s in range(1, 5):
            p = (F - 1) if (F + s) % 2 else (F - 1) // 2  # both extremes of the padding range over the grid
            I = 9 + F + 2 * s                              # several outputs per axis for every (F, s)
            out.append(Layer(f"g{F}{s}", 67, 24, I, I + 1, 40, F, F, s, s, p, p))
    return out


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("lay", _grid(), ids=lambda l: f"F{l.FH}s{l.sh}p{l.ph}")
def test_filter_stride_grid(torch_cuda, lay, dtype):
    check_full(torch_cuda, lay, dtype, config=19, idx=10 * lay.FH + lay.sh)


def _np(t, dtype):
    """device tensor (bf16 / fp32) -> the float64 values it holds."""
    return t.detach().float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_dcgan_generator_step(torch_cuda, dtype):
    torch = torch_cuda
    from paper_2306_15951_b200 import ops as K
    N = 6
    # conv-layer view (X = the big side): generator layer k maps z_k (O_C channels,
    # OH x OW) to y_k (I_C channels, H x W)
    lays = [Layer("G4to8", N, 512, 8, 8, 1024, 4, 4, 2, 2, 1, 1),
            Layer("G8to16", N, 256, 16, 16, 512, 4, 4, 2, 2, 1, 1),
            Layer("G16to32", N, 128, 32, 32, 256, 4, 4, 2, 2, 1, 1),
            Layer("G32to64", N, 3, 64, 64, 128, 4, 4, 2, 2, 1, 1)]
    ins = [make_layer_inputs(l, 23, i, dtype) for i, l in enumerate(lays)]
    Ws = [dev(torch, a["W"], dtype).requires_grad_(True) for a in ins]
    z = dev(torch, ins[0]["dY"], dtype).requires_grad_(True)
    T = dev(torch, ins[-1]["X"], dtype)  # upstream gradient of the generated 64x64x3 image
    zs, ys = [], []
    h = z
    for l, w in zip(lays, Ws):
        zs.append(h)
        y = K.cks_conv_transpose2d(h, w, (l.H, l.W), (l.sh, l.sw), (l.ph, l.pw))
        y.retain_grad()
        ys.append(y)
        h = y.to(w.dtype)  # next layer's input in the input precision
        if h is not y:
            h.retain_grad()
    (ys[-1] * T.float()).sum().backward()
    torch.cuda.synchronize()
    for k, l in enumerate(lays):
        g = (l.sh, l.sw, l.ph, l.pw)
        zk = _np(zs[k], dtype)
        wk = _np(Ws[k].detach(), dtype)
        # forward: y_k = KS-deconv(z_k, W_k) on the z_k the chain produced
        check(_np(ys[k], dtype), O.deconv_ref(zk, wk, l.H, l.W, *g), dtype, f"{l.name} generator fwd",
              red_len(l, "deconv"))
        # backward: the wrapper rounds dL/dy_k to the input dtype before its kernels
        gy = ys[k].grad.to(Ws[k].dtype)
        gk = _np(gy, dtype)
        check(_np(Ws[k].grad, dtype), O.wgrad_ref(gk, zk, l.FH, l.FW, *g), dtype + "_grad",
              f"{l.name} generator dW", red_len(l, "wgrad"))
        dz = zs[k].grad
        check(_np(dz, dtype), O.conv_ref(gk, wk, *g), dtype + "_grad", f"{l.name} generator dz", red_len(l, "fwd"))
