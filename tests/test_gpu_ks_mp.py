"""GPU parity of the multi-phase KS-deconv for narrow outputs
(cks_deconv2d_ex(CKS_KS_MULTIPHASE)): with F % s == 0 every phase has the
same CH x CW sub-filter (Alg. 2 Stage1, Fig. 5), and shifting each
phase's row index by its a_y (T2, Alg. 2B) makes all phases read the same
dY window, so the sh*sw phases are stacked on the GEMM N dimension of one
unit-stride ConvV2 over dY, followed by the phase-strided scatter of Stage3
(P:186).  Against the fp64 oracle's zero-inserting definition (Eq 2)
and the Stage1 path."""
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


CASES = [Layer("mp_dcgan", 130, 3, 64, 64, 128, 4, 4, 2, 2, 1, 1),   # C4 G32to64 at reduced batch
         Layer("mp_odd", 67, 3, 13, 15, 40, 4, 4, 2, 2, 1, 1),      # odd extents: unread rows, ragged tiles
         Layer("mp_f2", 70, 5, 12, 12, 24, 2, 2, 2, 2, 0, 0),       # 2x2 s2: one tap per phase
         Layer("mp_f6s3", 33, 2, 20, 17, 64, 6, 6, 3, 3, 2, 2),     # 9 phases of 2x2
         Layer("mp_p0", 9, 8, 16, 16, 16, 4, 4, 2, 2, 0, 0),        # no padding, 8 outputs
         Layer("mp_f4s4", 20, 3, 16, 16, 32, 4, 4, 4, 4, 0, 0),     # 16 phases of 1x1
         Layer("mp_rect", 40, 4, 14, 20, 48, 4, 2, 2, 2, 1, 0)]     # different axes


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("lay", CASES, ids=lambda l: l.name)
def test_multiphase_ks_deconv(torch_cuda, lay, dtype):
    a, got = _deconv(torch_cuda, lay, dtype, 26, 0, "multiphase")
    ref = O.deconv_ref(a["dY"], a["W"], lay.H, lay.W, lay.sh, lay.sw, lay.ph, lay.pw)
    check(got, ref, dtype, f"{lay.name} multi-phase deconv", red_len(lay, "deconv"))
    _, s1 = _deconv(torch_cuda, lay, dtype, 26, 0, "stage1")
    check(got, s1, dtype, f"{lay.name} multi-phase vs stage1", red_len(lay, "deconv"))
    _, auto = _deconv(torch_cuda, lay, dtype, 26, 0, "auto")  # the library's choice for W given: this path
    np.testing.assert_array_equal(auto, got)


def test_multiphase_rejects_ineligible(torch_cuda):
    torch = torch_cuda
    from paper_2306_15951_b200 import _lib as L
    from paper_2306_15951_b200 import ops as K
    W = torch.zeros((8, 3, 3, 3), dtype=torch.bfloat16, device="cuda")   # F = 3, s = 2: unequal phases
    G = torch.zeros((2, 4, 4, 8), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(L.CksError):
        K.deconv2d(G, W, (8, 8), 2, 1, ks_mode="multiphase")
