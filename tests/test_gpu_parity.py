"""GPU parity: the CUDA path (through the C ABI of libcks.so) against the
fp64 CPU oracle on identical seeded inputs.

Tolerance: the contract (BASELINE.json north_star) is a normwise relative
error <= 2e-2 for BF16 and <= 5e-3 for TF32 (fp32 accumulation).  Because the
oracle receives exactly the bf16 values the GPU multiplies, the only BF16
error source is fp32 accumulation order, so the tests also enforce a much
tighter bound (tight_bf16) to catch a dropped or
duplicated boundary tap that a 2e-2 normwise bound could hide on large maps.
"""
import numpy as np
import pytest

import oracle as O
from cks_synth import Layer, bf16_bits, get_config, make_layer_inputs

pytestmark = pytest.mark.gpu

TOL = {"bf16": 2e-2, "tf32": 5e-3,
       # gradients returned in the input dtype by the autograd wrappers: one extra
       # rounding of the fp32 result to bf16 (u = 2^-9) / none for fp32
       "bf16_grad": 2e-2, "tf32_grad": 5e-3}
U32 = 2.0 ** -24  # fp32 unit roundoff


def tight_bf16(k: int) -> float:
    """Tight bound for bf16-exact inputs: fp32 (tensor-core) accumulation of k
    terms has a typical relative error ~ u*sqrt(k); 32x margin, measured worst
    case 12x at k = 3.2M (ResNet stem wgrad) -- DESIGN.md "Tolerances"."""
    return max(1e-6, 32.0 * U32 * np.sqrt(k))


def red_len(lay, op):
    OH, OW = lay.out_hw()
    return {"fwd": lay.FH * lay.FW * lay.C, "deconv": lay.FH * lay.FW * lay.OC, "wgrad": lay.N * OH * OW}[op]


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2306_15951_b200 import build
    build.build()
    return torch


def dev(torch, a, dtype):
    """numpy float32 (bf16-representable for 'bf16') -> CUDA tensor."""
    if dtype == "bf16":
        bits = torch.from_numpy(bf16_bits(a).view(np.int16))
        return bits.view(torch.bfloat16).cuda()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def nrm_err(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.linalg.norm(ref)
    return np.linalg.norm(got - ref) / (den if den > 0 else 1.0)


def check(got, ref, dtype, what, k=1):
    e = nrm_err(got, ref)
    assert e <= TOL[dtype], f"{what}: normwise error {e:.3e} > {TOL[dtype]}"
    if dtype == "bf16_grad":
        assert e <= 2.0 ** -8 + tight_bf16(k), f"{what}: normwise error {e:.3e} > bf16 output rounding bound"
    if dtype == "bf16":
        assert e <= tight_bf16(k), f"{what}: normwise error {e:.3e} > tight bound {tight_bf16(k):.2e}"
    return e


def run_all(torch, lay: Layer, dtype="bf16", config=0, idx=0, ops=("fwd", "deconv", "wgrad"), gz=0,
            via_split=False):
    from paper_2306_15951_b200 import ops as K
    a = make_layer_inputs(lay, config, idx, dtype)
    X, W, G = dev(torch, a["X"], dtype), dev(torch, a["W"], dtype), dev(torch, a["dY"], dtype)
    out = {}
    s, p = (lay.sh, lay.sw), (lay.ph, lay.pw)
    if "fwd" in ops:
        out["fwd"] = K.conv2d_fwd(X, W, s, p)
    if "deconv" in ops:
        if via_split:
            cp = K.ks_split(W, s)
            out["deconv"] = K.deconv2d(G, W, (lay.H, lay.W), s, p, c_packed=cp)
        else:
            out["deconv"] = K.deconv2d(G, W, (lay.H, lay.W), s, p)
    if "wgrad" in ops:
        out["wgrad"] = K.dilated_wgrad(X, G, (lay.FH, lay.FW), s, p, gz=gz)
    torch.cuda.synchronize()
    return a, {k: v.cpu().numpy() for k, v in out.items()}


def check_full(torch, lay, dtype="bf16", **kw):
    a, got = run_all(torch, lay, dtype, **kw)
    s = (lay.sh, lay.sw, lay.ph, lay.pw)
    if "fwd" in got:
        check(got["fwd"], O.conv_ref(a["X"], a["W"], *s), dtype, f"{lay} fwd", red_len(lay, "fwd"))
    if "deconv" in got:
        check(got["deconv"], O.deconv_ref(a["dY"], a["W"], lay.H, lay.W, *s), dtype, f"{lay} deconv",
              red_len(lay, "deconv"))
    if "wgrad" in got:
        check(got["wgrad"], O.wgrad_ref(a["X"], a["dY"], lay.FH, lay.FW, *s), dtype, f"{lay} wgrad",
              red_len(lay, "wgrad"))
    return got


# ------------------------------------------------------------------ C1
@pytest.mark.parametrize("dtype", ["bf16"])
def test_c1_all_ops(torch_cuda, dtype):
    lay = get_config(0)[1][0]
    got = check_full(torch_cuda, lay, dtype)
    # brute-force scalar loops too (C1 is tiny)
    a = make_layer_inputs(lay, 0, 0, dtype)
    s = (lay.sh, lay.sw, lay.ph, lay.pw)
    assert nrm_err(got["fwd"], O.brute_conv(a["X"], a["W"], *s)) < tight_bf16(red_len(lay, "fwd"))
    assert nrm_err(got["deconv"], O.brute_deconv(a["dY"], a["W"], lay.H, lay.W, *s)) < tight_bf16(red_len(lay, "deconv"))
    assert nrm_err(got["wgrad"], O.brute_wgrad(a["X"], a["dY"], lay.FH, lay.FW, *s)) < tight_bf16(red_len(lay, "wgrad"))


def test_c1_tf32_all_ops(torch_cuda):
    lay = get_config(0)[1][0]
    check_full(torch_cuda, lay, "tf32")


# ------------------------------------------------------- random geometries
def _rand_layers(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        FH, FW = int(rng.choice([1, 2, 3, 4, 5, 7])), int(rng.choice([1, 3, 4, 5]))
        sh, sw = int(rng.integers(1, 4)), int(rng.integers(1, 4))
        ph, pw = int(rng.integers(0, FH)), int(rng.integers(0, FW))
        H, W = int(rng.integers(max(1, FH - 2 * ph), 20)), int(rng.integers(max(1, FW - 2 * pw), 20))
        C = int(rng.choice([3, 8, 16, 24, 64, 72, 136]))
        OC = int(rng.choice([5, 8, 32, 64, 96, 200, 264]))
        N = int(rng.choice([1, 3, 130]))
        lay = Layer(f"rand{len(out)}", N, C, H, W, OC, FH, FW, sh, sw, ph, pw)
        try:
            O.geom(**lay.geom())
        except O.GeometryError:
            continue
        if N * H * W * max(C, OC) > 3e6:
            continue
        out.append(lay)
    return out


@pytest.mark.parametrize("lay", _rand_layers(24, 11), ids=lambda l: f"{l.N}x{l.H}x{l.W}x{l.C}-{l.OC}-f{l.FH}{l.FW}s{l.sh}{l.sw}p{l.ph}{l.pw}")
def test_random_geometries(torch_cuda, lay):
    check_full(torch_cuda, lay, "bf16", config=9, idx=int(lay.name[4:]))


@pytest.mark.parametrize("lay", _rand_layers(10, 23), ids=lambda l: f"tf32-{l.N}x{l.H}x{l.W}x{l.C}-{l.OC}-f{l.FH}{l.FW}s{l.sh}{l.sw}p{l.ph}{l.pw}")
def test_random_geometries_tf32(torch_cuda, lay):
    """TF32 (fp32 storage, TF32 tensor-core multiply): all three operators."""
    check_full(torch_cuda, lay, "tf32", config=8, idx=int(lay.name[4:]))


def _narrow_layers(n, seed, dtype="bf16"):
    """Narrow-channel layers (FW*C <= 64 bf16 / 32 fp32): the filter-row kernels
    (kernels/narrow.cuh); a few have a row pitch W*C*eb that is not a multiple
    of 16 bytes and take the padded per-tap path instead."""
    rng = np.random.default_rng(seed)
    out = []
    lim, align = (64, 8) if dtype == "bf16" else (32, 4)
    while len(out) < n:
        C = int(rng.choice([1, 2, 3, 4, 8, 16] if dtype == "bf16" else [1, 2, 3, 4, 8]))
        fws = [f for f in (1, 2, 3, 4, 5, 7) if f * C <= lim]
        if not fws:
            continue
        FW = int(rng.choice(fws))
        FH = int(rng.choice([1, 2, 3, 4, 5, 7]))
        sh, sw = int(rng.integers(1, 4)), int(rng.integers(1, 4))
        ph, pw = int(rng.integers(0, FH)), int(rng.integers(0, FW))
        H = int(rng.integers(max(1, FH - 2 * ph), 24))
        W = int(rng.integers(max(1, FW - 2 * pw), 24))
        if rng.random() < 0.8:  # mostly 16-byte row pitch (row path)
            q = align // np.gcd(align, C)
            W = max(q, (W + q - 1) // q * q)
        OC = int(rng.choice([5, 8, 32, 64, 96, 128, 200]))
        N = int(rng.choice([1, 63, 130, 257]))
        lay = Layer(f"narrow{len(out)}", N, C, H, W, OC, FH, FW, sh, sw, ph, pw)
        try:
            O.geom(**lay.geom())
        except O.GeometryError:
            continue
        if N * H * W * max(C, OC) > 4e6:
            continue
        out.append(lay)
    return out


@pytest.mark.parametrize("lay", _narrow_layers(20, 5), ids=lambda l: f"{l.N}x{l.H}x{l.W}x{l.C}-{l.OC}-f{l.FH}{l.FW}s{l.sh}{l.sw}p{l.ph}{l.pw}")
def test_narrow_channel_geometries(torch_cuda, lay):
    check_full(torch_cuda, lay, "bf16", config=7, idx=int(lay.name[6:]))


@pytest.mark.parametrize("lay", _narrow_layers(20, 17, "tf32"), ids=lambda l: f"tf32-{l.N}x{l.H}x{l.W}x{l.C}-{l.OC}-f{l.FH}{l.FW}s{l.sh}{l.sw}p{l.ph}{l.pw}")
def test_narrow_channel_geometries_tf32(torch_cuda, lay):
    """The filter-row kernels in TF32 (fp32 rows, kind::tf32; MN-major
    SWIZZLE_128B_BASE32B operands for Sk-dilated)."""
    check_full(torch_cuda, lay, "tf32", config=7, idx=100 + int(lay.name[6:]))


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("lay", [Layer("nb0", 5, 3, 6, 8, 8, 7, 7, 1, 1, 3, 3),     # windows overhang both sides
                                 Layer("nb1", 130, 3, 17, 24, 64, 5, 5, 1, 1, 2, 2),  # 2 border columns per side
                                 Layer("nb2", 67, 1, 12, 16, 8, 3, 3, 3, 3, 1, 1),    # stride 3, one channel
                                 Layer("nb3", 129, 4, 9, 12, 32, 7, 3, 2, 1, 6, 2),   # ph = FH - 1
                                 Layer("nb4", 64, 2, 20, 8, 40, 3, 7, 1, 2, 1, 6)],   # pw = FW - 1, s = (1, 2)
                         ids=lambda l: l.name)
def test_narrow_border_classes(torch_cuda, lay, dtype):
    """Border columns are classes of their own (left: box origin 0; right: the
    32-byte K-chunk grid ends at the row end); output rows trimmed to their
    valid filter rows; R-row tiles."""
    check_full(torch_cuda, lay, dtype, config=7, idx=200 + int(lay.name[2:]))


@pytest.mark.parametrize("gz", [1, 3, 200])
@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_narrow_wgrad_segments_dtypes(torch_cuda, gz, dtype):
    """Row-path Sk-dilated with explicit G_Z spread over the column
    classes: bit-identical on repeat, equal to the oracle."""
    lay = Layer("nz", 70, 3, 20, 16, 64, 7, 7, 2, 2, 3, 3)
    a, got = run_all(torch_cuda, lay, dtype, config=7, idx=98, ops=("wgrad",), gz=gz)
    _, got2 = run_all(torch_cuda, lay, dtype, config=7, idx=98, ops=("wgrad",), gz=gz)
    assert np.array_equal(got["wgrad"], got2["wgrad"])
    ref = O.wgrad_ref(a["X"], a["dY"], 7, 7, 2, 2, 3, 3)
    check(got["wgrad"], ref, dtype, f"narrow wgrad gz={gz}", red_len(lay, "wgrad"))


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("lay", [Layer("wf0", 20, 8, 128, 128, 32, 10, 10, 2, 2, 4, 4),
                                 Layer("wf1", 9, 3, 96, 224, 64, 11, 11, 2, 2, 5, 5)],
                         ids=lambda l: l.name)
def test_wide_filter_stride2_program_capacity(torch_cuda, lay, dtype):
    """Wide filters with stride > 1 on wide maps: one MMA-program entry per
    (pixel, tap), so the plan must narrow the pixel block to fit the 64-entry
    program lists (kernels/igemm.cuh kProgSlot)."""
    check_full(torch_cuda, lay, dtype, config=17, idx=int(lay.name[2:]), ops=("fwd",))


@pytest.mark.parametrize("lay", [Layer("sk0", 100, 512, 4, 4, 256, 3, 3, 2, 2, 1, 1),
                                 Layer("sk1", 70, 256, 5, 5, 512, 3, 3, 2, 2, 1, 1),
                                 Layer("sk2", 129, 384, 3, 3, 128, 3, 3, 1, 1, 1, 1)],
                         ids=lambda l: l.name)
def test_igemm_split_k_small_grid(torch_cuda, lay):
    """Under-filled grids (< 32 output tiles, >= 16 row steps) take the in-kernel
    deterministic split-K (Z = 2, last-arriving CTA sums the partials)."""
    check_full(torch_cuda, lay, "bf16", config=6, idx=int(lay.name[2:]))
    a, got = run_all(torch_cuda, lay, "bf16", config=6, idx=int(lay.name[2:]))
    _, again = run_all(torch_cuda, lay, "bf16", config=6, idx=int(lay.name[2:]))
    for op in got:
        assert np.array_equal(got[op], again[op]), f"{op} not deterministic"


def test_sharded_step_single_gpu(torch_cuda):
    """The batch-sharded arithmetic of dist.py on one GPU: two shards run
    sequentially, partial dW summed on the host == full-batch oracle."""
    torch = torch_cuda
    from paper_2306_15951_b200.dist import FlatGrads, shard_range, sharded_layer_step
    lay = Layer("sh", 131, 64, 9, 9, 96, 3, 3, 2, 2, 1, 1)
    a = make_layer_inputs(lay, 5, 0)
    X, W, G = dev(torch, a["X"], "bf16"), dev(torch, a["W"], "bf16"), dev(torch, a["dY"], "bf16")
    fg = FlatGrads([(lay.OC, lay.FH, lay.FW, lay.C)], "cuda")
    dW = np.zeros((lay.OC, lay.FH, lay.FW, lay.C))
    Ys, dXs = [], []
    for r in range(2):
        lo, hi = shard_range(lay.N, 2, r)
        y, dx = sharded_layer_step(X[lo:hi].contiguous(), W, G[lo:hi].contiguous(), (2, 2), (1, 1), fg.views[0])
        torch.cuda.synchronize()
        Ys.append(y.cpu().numpy())
        dXs.append(dx.cpu().numpy())
        dW += fg.views[0].cpu().numpy()
    s = (lay.sh, lay.sw, lay.ph, lay.pw)
    check(np.concatenate(Ys), O.conv_ref(a["X"], a["W"], *s), "bf16", "sharded fwd", red_len(lay, "fwd"))
    check(np.concatenate(dXs), O.deconv_ref(a["dY"], a["W"], lay.H, lay.W, *s), "bf16", "sharded deconv",
          red_len(lay, "deconv"))
    check(dW, O.wgrad_ref(a["X"], a["dY"], lay.FH, lay.FW, *s), "bf16", "sharded wgrad", red_len(lay, "wgrad"))


def test_empty_phase_and_unread_rows(torch_cuda):
    # 1x1 s2 downsample: KS phase y=1 has CH=0 -> odd rows of dX must be 0 (c11);
    # I=6, F=3, s=2, p=0: row 5 of X is never read -> dX row 5 = 0 (c10).
    for lay in (Layer("ds", 4, 64, 8, 8, 128, 1, 1, 2, 2, 0, 0), Layer("tail", 3, 16, 6, 7, 24, 3, 3, 2, 2, 0, 0)):
        got = check_full(torch_cuda, lay)
        if lay.name == "ds":
            assert np.all(got["deconv"][:, 1::2, :, :] == 0) and np.all(got["deconv"][:, :, 1::2, :] == 0)
        else:
            assert np.all(got["deconv"][:, 5, :, :] == 0)


def test_ks_split_exact_and_cached_path(torch_cuda):
    torch = torch_cuda
    from paper_2306_15951_b200 import ops as K
    lay = Layer("g", 5, 24, 8, 8, 40, 4, 4, 2, 2, 1, 1)
    a = make_layer_inputs(lay, 7, 0)
    W = dev(torch, a["W"], "bf16")
    cp = K.ks_split(W, (2, 2)).float().cpu().numpy()
    Ck, CH, CW = O.ks_split_alg(a["W"], 2, 2)          # [y, x, oc, ch, cw, ic]
    OCp = (lay.OC + 7) // 8 * 8
    CHm, CWm = Ck.shape[3], Ck.shape[4]
    cp = cp.reshape(2 * 2, lay.C, CHm * CWm, OCp)
    for y in range(2):
        for x in range(2):
            for ch in range(CHm):
                for cw in range(CWm):
                    np.testing.assert_array_equal(cp[y * 2 + x, :, ch * CWm + cw, :lay.OC], Ck[y, x, :, ch, cw, :].T)
    assert np.all(cp[..., lay.OC:] == 0)
    g1 = run_all(torch, lay, config=7, ops=("deconv",))[1]["deconv"]
    g2 = run_all(torch, lay, config=7, ops=("deconv",), via_split=True)[1]["deconv"]
    np.testing.assert_array_equal(g1, g2)


@pytest.mark.parametrize("gz", [1, 2, 3, 7])
def test_wgrad_gz_segments_deterministic(torch_cuda, gz):
    lay = Layer("w", 130, 64, 9, 9, 128, 3, 3, 2, 2, 1, 1)
    got = check_full(torch_cuda, lay, ops=("wgrad",), gz=gz)
    again = run_all(torch_cuda, lay, ops=("wgrad",), gz=gz)[1]["wgrad"]
    np.testing.assert_array_equal(got["wgrad"], again)


# ------------------------------------------- config layers, reduced batch
def _config_layers():
    out = []
    for cfg in (1, 2, 3, 5):
        for i, lay in enumerate(get_config(cfg)[1]):
            if lay.name.startswith(("l1_", "l2_", "l3_", "l4_")) and not lay.name.endswith("_0"):
                continue  # repeated shapes
            out.append((cfg, i, lay))
    return out


@pytest.mark.parametrize("cfg,i,lay", _config_layers(), ids=lambda v: v.name if isinstance(v, Layer) else str(v))
def test_config_layers_reduced_batch(torch_cuda, cfg, i, lay):
    """Each config layer at N=130 when the full layer is small enough for the
    oracle (spans 2 batch tiles + a ragged tail), else N=3."""
    big = lay.H * lay.W * max(lay.C, lay.OC) * lay.FH * lay.FW * lay.OC * lay.C
    n = 130 if big < 4e9 else 3
    check_full(torch_cuda, lay.with_batch(n), "bf16", config=cfg, idx=i, ops=lay.ops)


@pytest.mark.parametrize("cfg,i,lay", _config_layers()[::3], ids=lambda v: v.name if isinstance(v, Layer) else str(v))
def test_config_layers_reduced_batch_tf32(torch_cuda, cfg, i, lay):
    """Every third config layer in TF32 (fp32 storage), reduced batch as above."""
    big = lay.H * lay.W * max(lay.C, lay.OC) * lay.FH * lay.FW * lay.OC * lay.C
    n = 67 if big < 4e9 else 2
    check_full(torch_cuda, lay.with_batch(n), "tf32", config=cfg, idx=i, ops=lay.ops)


# ------------------------------------------ full size, sampled outputs
def _full_tf32():
    """TF32 at full size: EVERY distinct shape of the headline workload (C3 = C5 layers at
    N = 256: stem, l1, l2a / l2ds / l2, l3a / l3ds / l3, l4a / l4ds / l4 -- the plans the bench
    times: G_Z, clusters, CTA pairs, row tiles, row kernels) and the C4 generator layers."""
    keep = {"stem", "l1_0", "l2a", "l2ds", "l2_0", "l3a", "l3ds", "l3_0", "l4a", "l4ds", "l4_0"}
    return [c for c in _config_layers() if (c[0] == 2 and c[2].name in keep) or c[0] == 3]


@pytest.mark.parametrize("cfg,i,lay,dtype", [c + ("bf16",) for c in _config_layers() if c[0] in (1, 3, 5)][::2] +
                         [c + ("bf16",) for c in _config_layers() if c[0] == 2][::3] +
                         [c + ("tf32",) for c in _full_tf32()],
                         ids=lambda v: v.name if isinstance(v, Layer) else str(v))
def test_config_layers_full_size_sampled(torch_cuda, cfg, i, lay, dtype):
    """Full BASELINE batch, the bench's launch configuration; the oracle
    computes sampled outputs one by one (rows for fwd/deconv, taps for wgrad)."""
    a, got = run_all(torch_cuda, lay, dtype, config=cfg, idx=i, ops=lay.ops)
    rng = np.random.default_rng(cfg * 100 + i)
    s = (lay.sh, lay.sw, lay.ph, lay.pw)
    OH, OW = lay.out_hw()
    if "fwd" in got:
        smp = [(int(rng.integers(lay.N)), int(rng.integers(OH)), int(rng.integers(OW))) for _ in range(24)]
        smp += [(lay.N - 1, 0, 0), (0, OH - 1, OW - 1)]
        ref = O.conv_ref_rows(a["X"], a["W"], *s, smp)
        check(np.stack([got["fwd"][t] for t in smp]), ref, dtype, f"{lay.name} fwd sampled", red_len(lay, "fwd"))
    if "deconv" in got:
        smp = [(int(rng.integers(lay.N)), int(rng.integers(lay.H)), int(rng.integers(lay.W))) for _ in range(24)]
        smp += [(lay.N - 1, lay.H - 1, lay.W - 1), (0, 0, 0)]
        ref = O.deconv_ref_rows(a["dY"], a["W"], lay.H, lay.W, *s, smp)
        check(np.stack([got["deconv"][t] for t in smp]), ref, dtype, f"{lay.name} deconv sampled",
              red_len(lay, "deconv"))
    if "wgrad" in got:
        taps = [(0, 0), (lay.FH - 1, lay.FW - 1), (lay.FH // 2, lay.FW // 2)]
        ref = O.wgrad_ref_taps(a["X"], a["dY"], lay.FH, lay.FW, *s, taps)
        check(np.stack([got["wgrad"][:, fh, fw, :] for fh, fw in taps]), ref, dtype, f"{lay.name} wgrad sampled",
              red_len(lay, "wgrad"))


# ------------------------------------------ KB-ZINS (zero-inserted baseline)
def _zins_layers():
    lays = [get_config(0)[1][0],
            Layer("zds", 5, 64, 8, 8, 128, 1, 1, 2, 2, 0, 0),       # 1x1 s2: empty KS phase
            Layer("zdc", 7, 40, 8, 8, 24, 4, 4, 2, 2, 1, 1),        # DCGAN 4x4 s2 p1
            Layer("zt", 3, 16, 6, 7, 24, 3, 3, 2, 2, 0, 0),         # output padding r = 1
            Layer("zn", 9, 3, 16, 16, 64, 7, 7, 2, 2, 3, 3),        # narrow channels (row kernels)
            Layer("z3", 4, 24, 11, 13, 5, 5, 3, 3, 2, 2, 1)]        # s3, OC not a 16-byte multiple
    return lays + _rand_layers(6, 31)


@pytest.mark.parametrize("lay", _zins_layers(), ids=lambda l: f"{l.name}-{l.N}x{l.H}x{l.W}x{l.C}-{l.OC}-f{l.FH}{l.FW}s{l.sh}{l.sw}p{l.ph}{l.pw}")
@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_zins_formulation_matches_oracle(torch_cuda, lay, dtype):
    """cks_zins_*: the textbook zero-padding / zero-inserting formulation
    (Eqs (1)-(3) as written) on the same kernels equals the oracle --
    the extra terms are exact zeros."""
    torch = torch_cuda
    from paper_2306_15951_b200 import ops as K
    a = make_layer_inputs(lay, 12, 0, dtype)
    X, W, G = dev(torch, a["X"], dtype), dev(torch, a["W"], dtype), dev(torch, a["dY"], dtype)
    s, p = (lay.sh, lay.sw), (lay.ph, lay.pw)
    y = K.zins_conv2d_fwd(X, W, s, p)
    dx = K.zins_deconv2d(G, W, (lay.H, lay.W), s, p)
    dw = K.zins_wgrad(X, G, (lay.FH, lay.FW), s, p)
    torch.cuda.synchronize()
    g = (lay.sh, lay.sw, lay.ph, lay.pw)
    check(y.cpu().numpy(), O.conv_ref(a["X"], a["W"], *g), dtype, f"{lay} zins fwd", red_len(lay, "fwd"))
    check(dx.cpu().numpy(), O.deconv_ref(a["dY"], a["W"], lay.H, lay.W, *g), dtype, f"{lay} zins deconv",
          lay.FH * lay.FW * lay.OC)
    OH, OW = lay.out_hw()
    check(dw.cpu().numpy(), O.wgrad_ref(a["X"], a["dY"], lay.FH, lay.FW, *g), dtype, f"{lay} zins wgrad",
          lay.N * ((OH - 1) * lay.sh + 1) * ((OW - 1) * lay.sw + 1))


# ------------------------------------------------ autograd (conv-layer training)
@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_autograd_conv_layer(torch_cuda, dtype):
    """CKSConv2dFunction: loss = <conv(X, W), T>; autograd's dX, dW come from
    KS-deconv and Sk-dilated with dY = T -- checked against the
    oracle definitions."""
    torch = torch_cuda
    from paper_2306_15951_b200 import ops as K
    lay = Layer("ag", 131, 24, 11, 10, 40, 3, 3, 2, 2, 1, 1)
    a = make_layer_inputs(lay, 13, 0, dtype)
    X = dev(torch, a["X"], dtype).requires_grad_(True)
    W = dev(torch, a["W"], dtype).requires_grad_(True)
    T = dev(torch, a["dY"], dtype)
    y = K.cks_conv2d(X, W, 2, 1)
    (y * T.float()).sum().backward()
    torch.cuda.synchronize()
    g = (2, 2, 1, 1)
    check(y.detach().cpu().numpy(), O.conv_ref(a["X"], a["W"], *g), dtype, "autograd fwd", red_len(lay, "fwd"))
    check(X.grad.float().cpu().numpy(), O.deconv_ref(a["dY"], a["W"], lay.H, lay.W, *g), dtype + "_grad",
          "autograd dX", red_len(lay, "deconv"))
    check(W.grad.float().cpu().numpy(), O.wgrad_ref(a["X"], a["dY"], 3, 3, *g), dtype + "_grad", "autograd dW",
          red_len(lay, "wgrad"))


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_autograd_generator_layer(torch_cuda, dtype):
    """CKSConvTranspose2dFunction, a DCGAN generator layer (4x4 s2 p1):
    forward = KS-deconv of z; backward dz = ConvV2 of dY, dW = Sk-dilated(dY, z)."""
    torch = torch_cuda
    from paper_2306_15951_b200 import ops as K
    lay = Layer("gen", 70, 16, 16, 16, 64, 4, 4, 2, 2, 1, 1)   # conv view: X = the big side (16x16x16)
    a = make_layer_inputs(lay, 14, 0, dtype)
    Z = dev(torch, a["dY"], dtype).requires_grad_(True)        # generator input (8x8x64)
    W = dev(torch, a["W"], dtype).requires_grad_(True)
    T = dev(torch, a["X"], dtype)                              # upstream gradient of the 16x16x16 output
    y = K.cks_conv_transpose2d(Z, W, (16, 16), 2, 1)
    (y * T.float()).sum().backward()
    torch.cuda.synchronize()
    g = (2, 2, 1, 1)
    check(y.detach().cpu().numpy(), O.deconv_ref(a["dY"], a["W"], 16, 16, *g), dtype, "generator fwd",
          red_len(lay, "deconv"))
    check(Z.grad.float().cpu().numpy(), O.conv_ref(a["X"], a["W"], *g), dtype + "_grad", "generator dz",
          red_len(lay, "fwd"))
    check(W.grad.float().cpu().numpy(), O.wgrad_ref(a["X"], a["dY"], 4, 4, *g), dtype + "_grad", "generator dW",
          red_len(lay, "wgrad"))


# ------------------------------------- Sk-dilated row tiles (F_W taps per tile)
@pytest.mark.parametrize("lay,gz", [(Layer("rt0", 130, 64, 40, 40, 48, 3, 3, 1, 1, 1, 1), 0),
                                    (Layer("rt1", 130, 40, 40, 37, 64, 3, 3, 1, 1, 1, 1), 3),
                                    (Layer("rt2", 200, 64, 81, 80, 24, 3, 3, 2, 2, 1, 1), 0),
                                    (Layer("rt3", 130, 64, 40, 40, 64, 3, 3, 1, 1, 0, 0), 7),
                                    (Layer("rt4", 130, 64, 40, 40, 64, 5, 3, 1, 1, 2, 1), 1),
                                    (Layer("rt5", 130, 128, 30, 30, 96, 3, 3, 1, 1, 1, 1), 0),   # BN = 128 row tiles
                                    (Layer("rt6", 140, 112, 29, 31, 128, 3, 3, 1, 1, 1, 1), 5)],
                         ids=lambda v: v.name if isinstance(v, Layer) else f"gz{v}")
@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_wgrad_row_tiles(torch_cuda, lay, gz, dtype):
    """Large-map 3-wide filters with I_C <= 64 take the row-tile Sk-dilated
    kernel (one filter row's F_W taps per tile share the dY block, per-tap
    trimmed ow ranges, O_C <= 64 loads only the valid dY rows -- one bf16 /
    two tf32 atoms): against the oracle, for several G_Z segmentations,
    deterministic on repeat."""
    a, got = run_all(torch_cuda, lay, dtype, config=15, idx=int(lay.name[2:]), ops=("wgrad",), gz=gz)
    ref = O.wgrad_ref(a["X"], a["dY"], lay.FH, lay.FW, lay.sh, lay.sw, lay.ph, lay.pw)
    check(got["wgrad"], ref, dtype, f"{lay} row-tile wgrad gz={gz}", red_len(lay, "wgrad"))
    again = run_all(torch_cuda, lay, dtype, config=15, idx=int(lay.name[2:]), ops=("wgrad",), gz=gz)[1]["wgrad"]
    np.testing.assert_array_equal(got["wgrad"], again)


# ---------------------------------------------- CTA-pair (cta_group::2) tiles
@pytest.mark.parametrize("lay", [Layer("pr0", 300, 128, 14, 14, 256, 3, 3, 1, 1, 1, 1),
                                 Layer("pr1", 256, 256, 7, 9, 384, 3, 3, 1, 1, 1, 1),
                                 Layer("pr2", 260, 128, 15, 14, 512, 3, 3, 2, 2, 1, 1),
                                 Layer("pr3", 384, 512, 8, 8, 256, 4, 4, 2, 2, 1, 1)],
                         ids=lambda l: l.name)
@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_pair_tiles(torch_cuda, lay, dtype):
    """>= 256 output channels and > 128 images: 2-CTA tiles (M = 256 images of one
    pixel across a CTA pair, N = 256 channels, each CTA holding half of B); odd
    image-block counts leave the last pair's second CTA out of range.  Forward
    and KS-deconv (whose output channels are I_C) against the oracle."""
    check_full(torch_cuda, lay, dtype, config=16, idx=int(lay.name[2:]), ops=("fwd", "deconv"))


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("lay", [Layer("wq0", 128, 3, 125, 128, 64, 7, 7, 2, 2, 3, 3),   # stem-like, odd O_H
                                 Layer("wq1", 128, 3, 33, 40, 64, 3, 3, 1, 1, 1, 1)],    # 3x3 s1, odd O_H
                         ids=lambda l: l.name)
def test_narrow_wgrad_multi_row_kblocks(torch_cuda, lay, dtype):
    """KB-WGRAD-ROW with q > 1 output rows per k-block (one X box of F_H + s_h(q-1) rows shared by
    the q rows' M-blocks; the last k-block of an odd O_H carries fewer rows)."""
    from paper_2306_15951_b200 import _lib as L
    g = L.make_geom(lay.N, lay.C, lay.H, lay.W, lay.OC, lay.FH, lay.FW, lay.sh, lay.sw, lay.ph, lay.pw)
    d = L.plan_dict(g, L.CKS_BF16 if dtype == "bf16" else L.CKS_TF32, L.CKS_OP_WGRAD)
    assert d["kind"] == "row_wgrad" and int(d["q"]) >= 2, d
    check_full(torch_cuda, lay, dtype, config=16, idx=int(lay.name[2:]), ops=("wgrad",))
