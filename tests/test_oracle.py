"""Pins for the fp64 CPU oracle (oracle/cks_oracle.py) against things other
than itself: the paper's printed counts (Figs 4-8, Table III), the hand case,
hand-derived index tables, scalar brute force, the adjoint identity, central
finite differences, torch's fp64 CPU convolution routines and the s=1/F=1
matmul special case.  CPU only (``-m "not gpu"``)."""
import json
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _rand_case(rng, max_i=9):
    while True:
        FH, FW = int(rng.choice([1, 2, 3, 4, 5, 7])), int(rng.choice([1, 2, 3, 4, 5]))
        sh, sw = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        ph, pw = int(rng.integers(0, FH)), int(rng.integers(0, FW))
        H, W = int(rng.integers(1, max_i + 1)), int(rng.integers(1, max_i + 1))
        try:
            g = O.geom(N=int(rng.integers(1, 3)), C=int(rng.integers(1, 4)), H=H, W=W,
                       OC=int(rng.integers(1, 3)), FH=FH, FW=FW, sh=sh, sw=sw, ph=ph, pw=pw)
        except O.GeometryError:
            continue
        return g


def _tensors(rng, g):
    X = rng.uniform(-1, 1, (g.N, g.H, g.W, g.C))
    Wt = rng.uniform(-1, 1, (g.OC, g.FH, g.FW, g.C))
    G = rng.uniform(-1, 1, (g.N, g.OH, g.OW, g.OC))
    return X, Wt, G


# ---------------------------------------------------------------- hand case
def test_hand_case_1d():
    h = _load("hand_case_1d.json")
    X = np.array(h["X"], float).reshape(1, 4, 1, 1)
    Wt = np.array(h["W"], float).reshape(1, 2, 1, 1)
    G = np.array(h["dY"], float).reshape(1, 2, 1, 1)
    s, p = h["stride"], h["pad"]
    Y = O.conv_ref(X, Wt, s, 1, p, 0)
    dX = O.deconv_ref(G, Wt, 4, 1, s, 1, p, 0)
    dW = O.wgrad_ref(X, G, 2, 1, s, 1, p, 0)
    assert Y.ravel().tolist() == h["Y"]
    assert dX.ravel().tolist() == h["dX"]
    assert dW.ravel().tolist() == h["dW"]
    ip = h["inner_product"]
    assert np.vdot(Y, G) == ip and np.vdot(X, dX) == ip and np.vdot(Wt, dW) == ip


# ------------------------------------------------ paper's printed counts
def test_paper_complexity_counts():
    c = _load("paper_counts.json")
    g = O.geom(**c["geometry"])
    rng = np.random.default_rng(0)
    X, Wt, G = _tensors(rng, g)
    _, m_normal = O.convv2_alg(X, Wt, g.sh, g.sw, g.ph, g.pw, trim=False)
    _, m_v2 = O.convv2_alg(X, Wt, g.sh, g.sw, g.ph, g.pw, trim=True)
    assert 2 * m_normal == c["conv_normal"] and 2 * m_v2 == c["convv2"]
    Ck, CH, CW = O.ks_split_alg(Wt, g.sh, g.sw)
    _, k1 = O.ks_deconv_alg(G, Ck, CH, CW, g.H, g.W, g.sh, g.sw, g.ph, g.pw, trim=False)
    _, k2 = O.ks_deconv_alg(G, Ck, CH, CW, g.H, g.W, g.sh, g.sw, g.ph, g.pw, trim=True)
    assert 2 * k1 == c["ks_deconv"] and 2 * k2 == c["ks_deconv_v2"]
    _, s1 = O.sk_dilated_alg(X, G, g.FH, g.FW, g.sh, g.sw, g.ph, g.pw, trim=False)
    _, s2 = O.sk_dilated_alg(X, G, g.FH, g.FW, g.sh, g.sw, g.ph, g.pw, trim=True)
    assert 2 * s1 == c["sk_dilated"] and 2 * s2 == c["sk_dilated_v2"]
    cnt = O.op_counts(g)
    assert cnt["T_deconv"] == c["T_deconv"] and cnt["T_dilated"] == c["T_dilated"]
    assert cnt["T_conv"] == c["conv_normal"] and cnt["zero_free_flops"] == c["convv2"]
    # the (sh*sw) claims of P:178 / P:208
    assert cnt["T_deconv"] == g.sh * g.sw * c["ks_deconv"]
    assert cnt["T_dilated"] * g.OH * g.OW == c["sk_dilated"] * cnt["OHp"] * cnt["OWp"]


def test_fig5_split_extents():
    c = _load("paper_counts.json")
    Wt = np.arange(9, dtype=float).reshape(1, 3, 3, 1) + 1
    Ck, CH, CW = O.ks_split_alg(Wt, 2, 2)
    assert list(Ck.shape[:2]) + list(Ck.shape[3:5]) == c["fig5_C_spatial_shape"]
    for key, (eh, ew) in c["fig5_extents"].items():
        y, x = int(key[0]), int(key[1])
        assert (CH[y], CW[x]) == (eh, ew)
        # the (eh x ew) block holds exactly W's taps of phase (y,x), rotated
        blk = Ck[y, x, 0, :, :, 0]
        assert np.count_nonzero(blk) == eh * ew
        assert np.count_nonzero(blk[eh:, :]) == 0 and np.count_nonzero(blk[:, ew:]) == 0
    # rotation: C00[0,0] is the last phase-(0,0) tap W[2,2] (W^rot180)
    assert Ck[0, 0, 0, 0, 0, 0] == Wt[0, 2, 2, 0] and Ck[0, 0, 0, 1, 1, 0] == Wt[0, 0, 0, 0]
    assert Ck[1, 1, 0, 0, 0, 0] == Wt[0, 1, 1, 0]


def test_fig7_leaping_sequence():
    c = _load("paper_counts.json")
    g = O.geom(**c["geometry"])
    rng = np.random.default_rng(1)
    X, _, G = _tensors(rng, g)
    visit = (tuple(c["fig7_tap"]), [])
    O.sk_dilated_alg(X, G[:, :, :, :1], g.FH, g.FW, g.sh, g.sw, g.ph, g.pw, trim=True, visit=visit)
    assert [list(v) for v in visit[1]] == c["fig7_sequence"]


# ------------------------------------------------------------- tables
@pytest.mark.parametrize("ax", _load("axis_tables.json")["axes"], ids=lambda a: a["name"])
def test_axis_tables_golden(ax):
    I, F, s, p = ax["I"], ax["F"], ax["s"], ax["p"]
    assert O.out_extent(I, F, s, p) == ax["O"]
    assert O.axis_V(I, F, s, p) == ax["V"]
    assert [list(r) for r in O.table_T1(I, F, s, p)] == ax["T1"]
    assert [list(r) for r in O.table_T3(I, F, s, p)] == ax["T3"]
    t2 = O.table_T2(I, F, s, p)
    for ph_got, ph_exp in zip(t2, ax["T2"]):
        for k in ("y", "CH", "oph", "ih_s", "U", "a"):
            assert ph_got[k] == ph_exp[k], (k, ph_got, ph_exp)
        assert [list(r) for r in ph_got["rows"]] == ph_exp["rows"]
    assert [list(r) for r in O.table_T4(I, F, s, p)] == ax["T4"]


@pytest.mark.parametrize("ax", _load("axis_tables.json")["t4_axes"], ids=lambda a: a["name"])
def test_t4_trim_classes_golden(ax):
    """T4 (trim classes) on config-sized axes, hand-derived: a version
    that never merges equal neighbours, or merges unequal ones, fails."""
    I, F, s, p = ax["I"], ax["F"], ax["s"], ax["p"]
    assert O.out_extent(I, F, s, p) == ax["O"]
    assert [list(r) for r in O.table_T4(I, F, s, p)] == ax["T4"]


def _axis_grid():
    for I in range(1, 14):
        for F in range(1, 8):
            for s in range(1, 5):
                for p in range(0, F):
                    if I + 2 * p - F >= 0:
                        yield I, F, s, p


def test_table_invariants_grid():
    """Partition invariants over the 1-D grid I 1..13, F 1..7, s 1..4, p<F."""
    n = 0
    for I, F, s, p in _axis_grid():
        V = O.axis_V(I, F, s, p)
        O_ = O.out_extent(I, F, s, p)
        t1, t3, t2 = O.table_T1(I, F, s, p), O.table_T3(I, F, s, p), O.table_T2(I, F, s, p)
        assert sum(fe - fs for (_, _, fs, fe) in t1) == V
        assert sum(oe - os_ for (_, _, os_, oe) in t3) == V
        assert sum(ph["CH"] for ph in t2) == F                       # sum_y CH_y = F
        rows = sorted(r[1] for ph in t2 for r in ph["rows"])
        assert rows == list(range(I))                                # phases partition [0, I)
        assert sum(r[4] - r[3] for ph in t2 for r in ph["rows"]) == V
        for ph in t2:
            for (u, i, oh_s, cs, ce) in ph["rows"]:
                if ph["CH"]:
                    assert oh_s == u + ph["a"]
                for ch in range(cs, ce):                              # every kept tap is a valid pair
                    f = ph["y"] + (ph["oph"] - ch) * s
                    assert 0 <= f < F and 0 <= oh_s + ch < O_ and (oh_s + ch) * s + f - p == i
        runs = O.table_T4(I, F, s, p)
        assert runs[0][0] == 0 and runs[-1][1] == O_
        for a, b in zip(runs, runs[1:]):                             # contiguous and maximal
            assert a[1] == b[0] and (a[2], a[3]) != (b[2], b[3])
        assert sum((r[1] - r[0]) * (r[3] - r[2]) for r in runs) == V  # classes cover the valid pairs
        n += 1
    assert n > 1000


# ----------------------------------------------- operator definitions
def test_brute_force_tiny_grid():
    rng = np.random.default_rng(2)
    for _ in range(60):
        g = _rand_case(rng, max_i=7)
        X, Wt, G = _tensors(rng, g)
        np.testing.assert_allclose(O.conv_ref(X, Wt, g.sh, g.sw, g.ph, g.pw),
                                   O.brute_conv(X, Wt, g.sh, g.sw, g.ph, g.pw), rtol=0, atol=1e-12)
        np.testing.assert_allclose(O.deconv_ref(G, Wt, g.H, g.W, g.sh, g.sw, g.ph, g.pw),
                                   O.brute_deconv(G, Wt, g.H, g.W, g.sh, g.sw, g.ph, g.pw), rtol=0, atol=1e-12)
        np.testing.assert_allclose(O.wgrad_ref(X, G, g.FH, g.FW, g.sh, g.sw, g.ph, g.pw),
                                   O.brute_wgrad(X, G, g.FH, g.FW, g.sh, g.sw, g.ph, g.pw), rtol=0, atol=1e-12)


def test_adjoint_identity():
    """<conv(X,W),G> = <X,deconv(G,W)> = <W,wgrad(X,G)> (chain rule of Eq (1)-(3))."""
    rng = np.random.default_rng(3)
    for _ in range(150):
        g = _rand_case(rng, max_i=12)
        X, Wt, G = _tensors(rng, g)
        a = np.vdot(O.conv_ref(X, Wt, g.sh, g.sw, g.ph, g.pw), G)
        b = np.vdot(X, O.deconv_ref(G, Wt, g.H, g.W, g.sh, g.sw, g.ph, g.pw))
        c = np.vdot(Wt, O.wgrad_ref(X, G, g.FH, g.FW, g.sh, g.sw, g.ph, g.pw))
        scale = max(1.0, abs(a))
        assert abs(a - b) <= 1e-11 * scale and abs(a - c) <= 1e-11 * scale


def test_finite_differences():
    """L = 0.5*||conv(X,W) - T||^2: dL/dX = deconv(Y-T, W), dL/dW = wgrad(X, Y-T)."""
    rng = np.random.default_rng(4)
    g = O.geom(N=2, C=2, H=6, W=6, OC=3, FH=3, FW=3, sh=2, sw=2, ph=1, pw=1)
    X, Wt, T = _tensors(rng, g)

    def loss(X_, W_):
        return 0.5 * np.sum((O.conv_ref(X_, W_, g.sh, g.sw, g.ph, g.pw) - T) ** 2)

    G = O.conv_ref(X, Wt, g.sh, g.sw, g.ph, g.pw) - T
    dX = O.deconv_ref(G, Wt, g.H, g.W, g.sh, g.sw, g.ph, g.pw)
    dW = O.wgrad_ref(X, G, g.FH, g.FW, g.sh, g.sw, g.ph, g.pw)
    eps = 1e-5
    for idx in np.ndindex(*X.shape):
        Xp, Xm = X.copy(), X.copy()
        Xp[idx] += eps
        Xm[idx] -= eps
        assert abs((loss(Xp, Wt) - loss(Xm, Wt)) / (2 * eps) - dX[idx]) < 1e-6
    for idx in np.ndindex(*Wt.shape):
        Wp, Wm = Wt.copy(), Wt.copy()
        Wp[idx] += eps
        Wm[idx] -= eps
        assert abs((loss(X, Wp) - loss(X, Wm)) / (2 * eps) - dW[idx]) < 1e-6
    # negative control: a transposed dW fails the check (S:431 fault injection)
    bad = np.transpose(dW, (0, 2, 1, 3))
    assert np.max(np.abs(bad - dW)) > 1e-3


def test_torch_fp64_cpu_cross_check():
    torch = pytest.importorskip("torch")
    F = torch.nn.functional
    rng = np.random.default_rng(5)
    for _ in range(80):
        g = _rand_case(rng, max_i=12)
        X, Wt, G = _tensors(rng, g)
        Xt = torch.from_numpy(X).permute(0, 3, 1, 2)
        Wtt = torch.from_numpy(Wt).permute(0, 3, 1, 2)
        Gt = torch.from_numpy(G).permute(0, 3, 1, 2)
        Y = F.conv2d(Xt, Wtt, stride=(g.sh, g.sw), padding=(g.ph, g.pw)).permute(0, 2, 3, 1).numpy()
        dX = torch.nn.grad.conv2d_input(Xt.shape, Wtt, Gt, stride=(g.sh, g.sw),
                                        padding=(g.ph, g.pw)).permute(0, 2, 3, 1).numpy()
        dW = torch.nn.grad.conv2d_weight(Xt, Wtt.shape, Gt, stride=(g.sh, g.sw),
                                         padding=(g.ph, g.pw)).permute(0, 2, 3, 1).numpy()
        np.testing.assert_allclose(O.conv_ref(X, Wt, g.sh, g.sw, g.ph, g.pw), Y, rtol=0, atol=1e-12)
        np.testing.assert_allclose(O.deconv_ref(G, Wt, g.H, g.W, g.sh, g.sw, g.ph, g.pw), dX, rtol=0, atol=1e-12)
        np.testing.assert_allclose(O.wgrad_ref(X, G, g.FH, g.FW, g.sh, g.sw, g.ph, g.pw), dW, rtol=0, atol=1e-12)


def test_matmul_special_case():
    """s=1, F=1, p=0: all three operators reduce to plain matrix products."""
    rng = np.random.default_rng(6)
    X = rng.uniform(-1, 1, (3, 4, 5, 6))
    Wt = rng.uniform(-1, 1, (7, 1, 1, 6))
    G = rng.uniform(-1, 1, (3, 4, 5, 7))
    Xm, Wm, Gm = X.reshape(-1, 6), Wt.reshape(7, 6), G.reshape(-1, 7)
    np.testing.assert_allclose(O.conv_ref(X, Wt, 1, 1, 0, 0).reshape(-1, 7), Xm @ Wm.T, atol=1e-13)
    np.testing.assert_allclose(O.deconv_ref(G, Wt, 4, 5, 1, 1, 0, 0).reshape(-1, 6), Gm @ Wm, atol=1e-13)
    np.testing.assert_allclose(O.wgrad_ref(X, G, 1, 1, 1, 1, 0, 0).reshape(7, 6), Gm.T @ Xm, atol=1e-13)


def test_algorithms_equal_definitions():
    """Alg. 1 / 2 / 2B / 3 / 3B under readings c1-c6 equal the definitions, and
    their MAC counts equal the zero-free count (V2) -- pins the readings."""
    rng = np.random.default_rng(7)
    for _ in range(120):
        g = _rand_case(rng, max_i=10)
        X, Wt, G = _tensors(rng, g)
        cnt = O.op_counts(g)
        Y, m1 = O.convv2_alg(X, Wt, g.sh, g.sw, g.ph, g.pw)
        np.testing.assert_allclose(Y, O.conv_ref(X, Wt, g.sh, g.sw, g.ph, g.pw), atol=1e-12)
        Ck, CH, CW = O.ks_split_alg(Wt, g.sh, g.sw)
        assert sum(CH) == g.FH and sum(CW) == g.FW
        dX, m2 = O.ks_deconv_alg(G, Ck, CH, CW, g.H, g.W, g.sh, g.sw, g.ph, g.pw)
        np.testing.assert_allclose(dX, O.deconv_ref(G, Wt, g.H, g.W, g.sh, g.sw, g.ph, g.pw), atol=1e-12)
        dX1, k1 = O.ks_deconv_alg(G, Ck, CH, CW, g.H, g.W, g.sh, g.sw, g.ph, g.pw, trim=False)
        np.testing.assert_allclose(dX1, dX, atol=1e-12)
        dW, m3 = O.sk_dilated_alg(X, G, g.FH, g.FW, g.sh, g.sw, g.ph, g.pw)
        np.testing.assert_allclose(dW, O.wgrad_ref(X, G, g.FH, g.FW, g.sh, g.sw, g.ph, g.pw), atol=1e-12)
        dW1, s1 = O.sk_dilated_alg(X, G, g.FH, g.FW, g.sh, g.sw, g.ph, g.pw, trim=False)
        np.testing.assert_allclose(dW1, dW, atol=1e-12)
        assert m1 == m2 == m3 == cnt["zero_free_macs"]
        # KS-V1 = zero-inserted / (sh*sw) exactly when I % s == 0
        if g.H % g.sh == 0 and g.W % g.sw == 0:
            assert k1 * g.sh * g.sw == cnt["T_deconv"] // 2
        # Sk-V1 = zero-inserted * (O_H O_W)/(O_H^p O_W^p) exactly
        assert s1 * cnt["OHp"] * cnt["OWp"] == (cnt["T_dilated"] // 2) * g.OH * g.OW


def test_samplers_match_full():
    rng = np.random.default_rng(8)
    g = O.geom(N=3, C=5, H=9, W=7, OC=4, FH=3, FW=2, sh=2, sw=1, ph=1, pw=1)
    X, Wt, G = _tensors(rng, g)
    Y = O.conv_ref(X, Wt, g.sh, g.sw, g.ph, g.pw)
    dX = O.deconv_ref(G, Wt, g.H, g.W, g.sh, g.sw, g.ph, g.pw)
    dW = O.wgrad_ref(X, G, g.FH, g.FW, g.sh, g.sw, g.ph, g.pw)
    ys = [(0, 0, 0), (2, g.OH - 1, g.OW - 1), (1, 2, 3)]
    np.testing.assert_allclose(O.conv_ref_rows(X, Wt, g.sh, g.sw, g.ph, g.pw, ys),
                               np.stack([Y[s] for s in ys]), atol=1e-12)
    xs = [(0, 0, 0), (2, g.H - 1, g.W - 1), (1, 4, 3)]
    np.testing.assert_allclose(O.deconv_ref_rows(G, Wt, g.H, g.W, g.sh, g.sw, g.ph, g.pw, xs),
                               np.stack([dX[s] for s in xs]), atol=1e-12)
    taps = [(0, 0), (2, 1)]
    got = O.wgrad_ref_taps(X, G, g.FH, g.FW, g.sh, g.sw, g.ph, g.pw, taps, n_chunk=2)
    np.testing.assert_allclose(got, np.stack([dW[:, a, b, :] for a, b in taps]), atol=1e-12)


def test_geometry_errors():
    with pytest.raises(O.GeometryError):
        O.out_extent(1, 3, 1, 0)        # filter larger than padded input
    with pytest.raises(O.GeometryError):
        O.out_extent(8, 3, 1, 3)        # p >= F (reading c16)
    assert O.out_extent(5, 3, 3, 1) == 2 and O.out_extent(4, 2, 2, 0) == 2
