"""GPU parity for ROW GROUPS (small per-GPU batches, N <= 64): the implicit
GEMM's M = 128 rows hold 128 / rg_ni consecutive output rows x rg_ni images
(rg_ni = 32 / 64) instead of 128 images of one pixel (DESIGN.md §7 "Row
groups").  Every group shares one trimmed window
(P:156), so these tests cover: groups cut by the border trim classes, ragged
last groups (fewer rows than rg_ph), batches that do not fill rg_ni, forward
strides 1-4 (the TMA element stride of the A box), KS-deconv phases (Stage1 /
Stage1-free / multi-phase), split-K tiles, and the C5 ResNet-18 layers at
32 images per GPU (C5 strong scaling on 8 GPUs)."""
import numpy as np
import pytest

import oracle as O
from cks_synth import Layer, get_config, make_layer_inputs
from test_gpu_parity import check, check_full, dev, red_len, run_all, torch_cuda  # noqa: F401

pytestmark = pytest.mark.gpu


def _rg_layers(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        FH, FW = int(rng.choice([1, 2, 3, 4, 5, 7])), int(rng.choice([1, 3, 4, 5]))
        sh, sw = int(rng.integers(1, 5)), int(rng.integers(1, 4))
        ph, pw = int(rng.integers(0, FH)), int(rng.integers(0, FW))
        H, W = int(rng.integers(max(1, FH - 2 * ph), 41)), int(rng.integers(max(1, FW - 2 * pw), 24))
        C = int(rng.choice([8, 16, 64, 72, 136]))
        OC = int(rng.choice([8, 32, 64, 96, 200]))
        N = int(rng.choice([1, 2, 7, 17, 31, 32, 33, 48, 63, 64]))
        lay = Layer(f"rg{len(out)}", N, C, H, W, OC, FH, FW, sh, sw, ph, pw)
        try:
            O.geom(**lay.geom())
        except O.GeometryError:
            continue
        if N * H * W * max(C, OC) > 3e6:
            continue
        out.append(lay)
    return out


def _id(l):
    return f"{l.N}x{l.H}x{l.W}x{l.C}-{l.OC}-f{l.FH}{l.FW}s{l.sh}{l.sw}p{l.ph}{l.pw}"


def _plan(lay, op, dtype="bf16"):
    from paper_2306_15951_b200 import _lib as L
    g = L.make_geom(lay.N, lay.C, lay.H, lay.W, lay.OC, lay.FH, lay.FW, lay.sh, lay.sw, lay.ph, lay.pw)
    dt = L.CKS_BF16 if dtype == "bf16" else L.CKS_TF32
    return L.plan_dict(g, dt, {"fwd": L.CKS_OP_FWD, "deconv": L.CKS_OP_DECONV}[op])


@pytest.mark.parametrize("lay", _rg_layers(28, 101), ids=_id)
def test_row_group_random_geometries(torch_cuda, lay):
    check_full(torch_cuda, lay, "bf16", config=11, idx=int(lay.name[2:]))


@pytest.mark.parametrize("lay", _rg_layers(14, 202), ids=lambda l: "tf32-" + _id(l))
def test_row_group_random_geometries_tf32(torch_cuda, lay):
    check_full(torch_cuda, lay, "tf32", config=12, idx=int(lay.name[2:]))


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("mode", ["stage1", "stage1_free"])
@pytest.mark.parametrize("lay", [Layer("rgk0", 20, 64, 29, 17, 64, 3, 3, 2, 2, 1, 1),
                                 Layer("rgk1", 40, 32, 30, 12, 64, 4, 4, 2, 2, 1, 1),
                                 Layer("rgk2", 9, 64, 33, 9, 32, 5, 3, 3, 1, 2, 1),
                                 Layer("rgk3", 64, 64, 16, 16, 128, 1, 1, 2, 2, 0, 0)], ids=lambda l: l.name)
def test_row_group_ks_modes(torch_cuda, lay, mode, dtype):
    """KS-deconv with row groups through both B-operand forms (packed sub-filters / W read directly):
    a group is a run of one phase's rows (A rows step 1, dX rows step s_h)."""
    from paper_2306_15951_b200 import ops as K
    a = make_layer_inputs(lay, 13, int(lay.name[3:]), dtype)
    G, W = dev(torch_cuda, a["dY"], dtype), dev(torch_cuda, a["W"], dtype)
    s, p = (lay.sh, lay.sw), (lay.ph, lay.pw)
    try:
        got = K.deconv2d(G, W, (lay.H, lay.W), s, p, ks_mode=mode)
    except Exception as e:  # Stage1-free needs IC rows of 16-byte multiples etc.
        if mode == "stage1_free" and "unsupported" in str(e).lower():
            pytest.skip("Stage1-free not eligible")
        raise
    torch_cuda.cuda.synchronize()
    ref = O.deconv_ref(a["dY"], a["W"], lay.H, lay.W, *s, lay.ph, lay.pw)
    check(got.cpu().numpy(), ref, dtype, f"{lay} deconv {mode}", red_len(lay, "deconv"))
    assert int(_plan(lay, "deconv", dtype)["rg"]) == (32 if lay.N <= 32 else 64)


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_row_group_multiphase_narrow_output(torch_cuda, dtype):
    """Narrow-output KS-deconv (phases stacked on N of one ConvV2 over dY) at a small batch."""
    lay = Layer("rgmp", 24, 3, 32, 32, 64, 4, 4, 2, 2, 1, 1)
    check_full(torch_cuda, lay, dtype, config=13, idx=9, ops=("deconv",))


def _c5_small(N):
    return [l.with_batch(N) for l in get_config(4)[1]]


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("lay", _c5_small(32), ids=lambda l: l.name)
def test_c5_layers_32_images(torch_cuda, lay, dtype):
    """C5 (ResNet-18 conv layers) at 32 images per GPU: fwd / KS-deconv / Sk-dilated against the
    oracle on sampled outputs (rows for fwd / deconv, taps for wgrad)."""
    a, got = run_all(torch_cuda, lay, dtype, config=4, idx=hash(lay.name) % 97, ops=lay.ops)
    rng = np.random.default_rng(len(lay.name))
    s = (lay.sh, lay.sw, lay.ph, lay.pw)
    OH, OW = lay.out_hw()
    if "fwd" in got:
        smp = [(int(rng.integers(lay.N)), int(rng.integers(OH)), int(rng.integers(OW))) for _ in range(24)]
        smp += [(lay.N - 1, 0, 0), (0, OH - 1, OW - 1), (lay.N - 1, OH - 1, 0)]
        ref = O.conv_ref_rows(a["X"], a["W"], *s, smp)
        check(np.stack([got["fwd"][t] for t in smp]), ref, dtype, f"{lay.name} fwd", red_len(lay, "fwd"))
    if "deconv" in got:
        smp = [(int(rng.integers(lay.N)), int(rng.integers(lay.H)), int(rng.integers(lay.W))) for _ in range(24)]
        smp += [(lay.N - 1, lay.H - 1, lay.W - 1), (0, 0, 0), (0, lay.H - 1, 0)]
        ref = O.deconv_ref_rows(a["dY"], a["W"], lay.H, lay.W, *s, smp)
        check(np.stack([got["deconv"][t] for t in smp]), ref, dtype, f"{lay.name} deconv", red_len(lay, "deconv"))
    if "wgrad" in got:
        taps = [(0, 0), (lay.FH - 1, lay.FW - 1), (lay.FH // 2, lay.FW // 2)]
        ref = O.wgrad_ref_taps(a["X"], a["dY"], lay.FH, lay.FW, *s, taps)
        check(np.stack([got["wgrad"][:, fh, fw, :] for fh, fw in taps]), ref, dtype, f"{lay.name} wgrad",
              red_len(lay, "wgrad"))


@pytest.mark.parametrize("N", [5, 32, 64])
def test_row_groups_leave_other_rows_untouched(torch_cuda, N):
    """Rows of a ragged last group beyond its length, and images beyond N, are computed in the
    tile but never stored: an output buffer pre-filled with NaN is fully overwritten and
    nothing outside it is written (guard band)."""
    from paper_2306_15951_b200 import ops as K
    torch = torch_cuda
    lay = Layer("rgg", N, 64, 23, 19, 64, 3, 3, 1, 1, 1, 1)
    a = make_layer_inputs(lay, 14, 0, "bf16")
    X, W = dev(torch, a["X"], "bf16"), dev(torch, a["W"], "bf16")
    OH, OW = lay.out_hw()
    n = N * OH * OW * lay.OC
    buf = torch.full((n + 4096,), float("nan"), device="cuda")
    y = buf[:n].view(N, OH, OW, lay.OC)
    K.conv2d_fwd(X, W, 1, 1, out=y)
    torch.cuda.synchronize()
    assert not torch.isnan(y).any()
    assert torch.isnan(buf[n:]).all()
    check(y.cpu().numpy(), O.conv_ref(a["X"], a["W"], 1, 1, 1, 1), "bf16", "rg guard", red_len(lay, "fwd"))


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("gz", [0, 1, 5])
@pytest.mark.parametrize("lay", [Layer("rgw0", 16, 64, 57, 45, 64, 3, 3, 1, 1, 1, 1),    # row tiles, odd widths
                                 Layer("rgw1", 32, 64, 41, 39, 64, 3, 3, 1, 2, 1, 1),    # s_w = 2 leaping chunks
                                 Layer("rgw2", 7, 128, 20, 23, 96, 3, 3, 2, 2, 1, 1),    # BN = 128, s = 2
                                 Layer("rgw3", 24, 96, 13, 17, 136, 5, 4, 1, 3, 2, 1),   # wide taps, s_w = 3
                                 Layer("rgw4", 3, 256, 9, 9, 256, 3, 3, 1, 1, 1, 1)],    # BN = 256, tiny batch
                         ids=lambda l: l.name)
def test_row_group_wgrad(torch_cuda, lay, gz, dtype):
    """Sk-dilated with position chunks: every tap multiplies only the K rows of its valid positions
    (chunks cut by the T3 ranges at both ends), G_Z segments split the chunk sequence."""
    check_full(torch_cuda, lay, dtype, config=15, idx=int(lay.name[3:]), ops=("wgrad",), gz=gz)


def _narrow_rg_layers(n, seed, dtype):
    """Narrow-channel ConvV2 (filter-row kernel) at small batches: row groups of rg_pc class
    columns x rg images, one box of the class's own tensor map (column stride cstep*sw*C)."""
    from test_gpu_parity import _narrow_layers
    out = []
    rng = np.random.default_rng(seed + 7)
    for lay in _narrow_layers(3 * n, seed, dtype):
        N = int(rng.choice([1, 5, 20, 32, 33, 47, 64]))
        out.append(Layer(lay.name.replace("narrow", "nrg"), N, lay.C, lay.H, lay.W + 8 * int(rng.integers(0, 3)),
                         lay.OC, lay.FH, lay.FW, lay.sh, lay.sw, lay.ph, lay.pw))
        if len(out) == n:
            break
    return out


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("k", range(14))
def test_row_group_narrow_fwd(torch_cuda, k, dtype):
    lay = _narrow_rg_layers(14, 41 if dtype == "bf16" else 43, dtype)[k]
    check_full(torch_cuda, lay, dtype, config=17, idx=k, ops=("fwd",))


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("lay", [Layer("nrs0", 32, 3, 61, 64, 64, 7, 7, 2, 2, 3, 3),    # ResNet stem at 32 images
                                 Layer("nrs1", 48, 3, 33, 40, 64, 3, 3, 1, 1, 1, 1),    # 3x3 s1, ragged groups
                                 Layer("nrs2", 7, 3, 32, 32, 64, 5, 5, 2, 2, 2, 2)],    # 5x5 s2, 7 images
                         ids=lambda l: l.name)
def test_row_group_narrow_fwd_plans(torch_cuda, lay, dtype):
    """The plan takes row groups for the filter-row ConvV2 and the output matches the oracle;
    a NaN-prefilled output proves every valid (image, pixel) is written and nothing else."""
    from paper_2306_15951_b200 import _lib as L
    from paper_2306_15951_b200 import ops as K
    torch = torch_cuda
    g = L.make_geom(lay.N, lay.C, lay.H, lay.W, lay.OC, lay.FH, lay.FW, lay.sh, lay.sw, lay.ph, lay.pw)
    d = L.plan_dict(g, L.CKS_BF16 if dtype == "bf16" else L.CKS_TF32, L.CKS_OP_FWD)
    assert d["kind"] == "row_fwd" and int(d["rg"]) == (32 if lay.N <= 32 else 64), d
    a = make_layer_inputs(lay, 18, int(lay.name[3:]), dtype)
    X, W = dev(torch, a["X"], dtype), dev(torch, a["W"], dtype)
    OH, OW = lay.out_hw()
    n = lay.N * OH * OW * lay.OC
    buf = torch.full((n + 4096,), float("nan"), device="cuda")
    y = buf[:n].view(lay.N, OH, OW, lay.OC)
    K.conv2d_fwd(X, W, (lay.sh, lay.sw), (lay.ph, lay.pw), out=y)
    torch.cuda.synchronize()
    assert not torch.isnan(y).any() and torch.isnan(buf[n:]).all()
    check(y.cpu().numpy(), O.conv_ref(a["X"], a["W"], lay.sh, lay.sw, lay.ph, lay.pw), dtype, f"{lay} fwd",
          red_len(lay, "fwd"))


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("gz", [0, 3])
@pytest.mark.parametrize("k", range(10))
def test_row_group_narrow_wgrad(torch_cuda, k, gz, dtype):
    """Narrow-channel Sk-dilated (filter-row kernel) at N <= 32: k-blocks of rg_pc class columns x
    rg images through per-class X / dY maps; columns past a class end are zero fill."""
    lay = _narrow_rg_layers(10, 51 if dtype == "bf16" else 53, dtype)[k]
    lay = Layer(lay.name, min(lay.N, 1 + (k * 7) % 32), lay.C, lay.H, lay.W, lay.OC, lay.FH, lay.FW, lay.sh,
                lay.sw, lay.ph, lay.pw)
    check_full(torch_cuda, lay, dtype, config=19, idx=k, ops=("wgrad",), gz=gz)


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_row_group_narrow_wgrad_stem(torch_cuda, dtype):
    from paper_2306_15951_b200 import _lib as L
    lay = Layer("nws0", 24, 3, 61, 64, 64, 7, 7, 2, 2, 3, 3)
    g = L.make_geom(lay.N, lay.C, lay.H, lay.W, lay.OC, lay.FH, lay.FW, lay.sh, lay.sw, lay.ph, lay.pw)
    d = L.plan_dict(g, L.CKS_BF16 if dtype == "bf16" else L.CKS_TF32, L.CKS_OP_WGRAD)
    assert d["kind"] == "row_wgrad" and int(d["rg"]) == 32, d
    check_full(torch_cuda, lay, dtype, config=19, idx=99, ops=("wgrad",))


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("lay", [Layer("rgz0", 16, 512, 4, 4, 256, 3, 3, 2, 2, 1, 1),    # cluster split-K (Z = 8)
                                 Layer("rgz1", 32, 512, 4, 4, 512, 3, 3, 1, 1, 1, 1),
                                 Layer("rgz2", 8, 256, 8, 8, 256, 3, 3, 1, 1, 1, 1),     # TF32: Z = 2 clusters
                                 Layer("rgz3", 64, 512, 7, 7, 512, 3, 3, 1, 1, 1, 1)],   # 2-row groups, l4-like
                         ids=lambda l: l.name)
def test_row_group_split_k(torch_cuda, lay, dtype):
    """Row groups with the in-cluster split-K reduce (DSMEM): the reducing CTA maps its column
    slice's rows back to (image, output row) of the group."""
    check_full(torch_cuda, lay, dtype, config=20, idx=int(lay.name[3:]))
