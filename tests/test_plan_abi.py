"""CPU-side checks of the C ABI (libcks.so): the library loads and exports
every symbol include/cks.h declares; the integer plan tables the kernels
consume are bit-exact against the oracle's brute-force enumeration; op
counts, validation and error codes.  No compute call is made (no GPU here)."""
import ctypes
import os
import re
import sys

import numpy as np
import pytest

import oracle as O
from paper_2306_15951_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2306_15951_b200 import build
    build.build()


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "cks.h")).read()
    declared = set(re.findall(r"^\s*(?:cks_status|const char\*|int)\s+(cks_\w+)\s*\(", hdr, re.M))
    assert declared == set(L.EXPORTS), declared ^ set(L.EXPORTS)
    lib = ctypes.CDLL(L.LIB_PATH)
    for name in declared:
        assert getattr(lib, name) is not None
    assert L.cks_version() >= 1


def _grid():
    for I in range(1, 14):
        for F in range(1, 8):
            for s in range(1, 5):
                for p in range(0, F):
                    if I + 2 * p - F >= 0:
                        yield I, F, s, p


def _flat_t2(phases):
    out = []
    for ph in phases:
        out += [ph["y"], ph["CH"], ph["oph"], ph["ih_s"], ph["U"], ph["a"]]
        for r in ph["rows"]:
            out += list(r)
    return out


def test_axis_tables_bit_exact_vs_oracle_grid():
    n = 0
    for I, F, s, p in _grid():
        assert L.cks_axis_table(I, F, s, p, 1) == [v for r in O.table_T1(I, F, s, p) for v in r], (I, F, s, p)
        assert L.cks_axis_table(I, F, s, p, 2) == _flat_t2(O.table_T2(I, F, s, p)), (I, F, s, p)
        assert L.cks_axis_table(I, F, s, p, 3) == [v for r in O.table_T3(I, F, s, p) for v in r], (I, F, s, p)
        assert L.cks_axis_table(I, F, s, p, 4) == [v for r in O.table_T4(I, F, s, p) for v in r], (I, F, s, p)
        n += 1
    assert n >= 1320


@pytest.mark.parametrize("I,F,s,p", [(224, 7, 2, 3), (56, 3, 2, 1), (56, 1, 2, 0), (64, 4, 2, 1), (7, 3, 1, 1),
                                     (4, 3, 2, 1), (255, 5, 3, 2)])
def test_axis_tables_config_sizes(I, F, s, p):
    assert L.cks_axis_table(I, F, s, p, 1) == [v for r in O.table_T1(I, F, s, p) for v in r]
    assert L.cks_axis_table(I, F, s, p, 2) == _flat_t2(O.table_T2(I, F, s, p))
    assert L.cks_axis_table(I, F, s, p, 3) == [v for r in O.table_T3(I, F, s, p) for v in r]


def test_op_counts_vs_oracle():
    from cks_synth import get_config
    for cfg in (0, 1, 2, 3):
        for lay in get_config(cfg)[1]:
            g = L.make_geom(lay.N, lay.C, lay.H, lay.W, lay.OC, lay.FH, lay.FW, lay.sh, lay.sw, lay.ph, lay.pw)
            got = L.cks_op_counts(g)
            ref = O.op_counts(O.geom(**lay.geom()))
            for k in ("zero_free_macs", "VH", "VW"):
                assert got[k] == ref[k], (lay.name, k)
            assert got["T_conv"] == ref["T_conv"] and got["T_deconv"] == ref["T_deconv"]
            assert got["T_dilated"] == ref["T_dilated"]
            assert L.cks_output_shape(g) == lay.out_hw()


def test_validation_errors():
    bad = [L.make_geom(1, 4, 1, 8, 8, 3, 3, 1, 1, 0, 0),   # F > padded I
           L.make_geom(1, 4, 8, 8, 8, 3, 3, 1, 1, 3, 1),   # p >= F
           L.make_geom(1, 4, 8, 8, 8, 3, 3, 0, 1, 1, 1),   # stride 0
           L.make_geom(0, 4, 8, 8, 8, 3, 3, 1, 1, 1, 1)]   # N = 0
    for g in bad:
        with pytest.raises(L.CksError) as e:
            L.cks_workspace_size(g, L.CKS_BF16, L.CKS_OP_FWD)
        assert e.value.status == 2
    g = L.make_geom(1, 4, 8, 8, 8, 3, 3, 1, 1, 1, 1, dh=2, dw=1)
    with pytest.raises(L.CksError) as e:
        L.cks_workspace_size(g, L.CKS_BF16, L.CKS_OP_FWD)
    assert e.value.status == 3
    # NULL / misaligned pointers are rejected before any CUDA call
    g = L.make_geom(2, 8, 8, 8, 8, 3, 3, 2, 2, 1, 1)
    lib = L.lib()
    assert lib.cks_conv2d_fwd(ctypes.byref(g), 1, None, None, None, None, 0, None) == 1
    assert lib.cks_conv2d_fwd(ctypes.byref(g), 1, 16, 17, 32, None, 0, None) == 4
    assert lib.cks_deconv2d(ctypes.byref(g), 1, 16, 16, 16, 16, None, 0, None) == 1   # both w and c_packed
    assert lib.cks_dilated_wgrad(ctypes.byref(g), 1, 16, 16, 16, -1, None, 0, None) == 3
    # capacity error for tables
    n = ctypes.c_size_t()
    buf = (ctypes.c_int64 * 2)()
    assert lib.cks_axis_table(8, 3, 2, 1, 1, buf, 2, ctypes.byref(n)) == 7 and n.value == 16


def test_workspace_and_launch_counts():
    g = L.make_geom(128, 3, 32, 33, 64, 3, 3, 1, 1, 1, 1)   # I_C = 3, odd row pitch -> padded staging
    assert L.cks_workspace_size(g, L.CKS_BF16, L.CKS_OP_FWD) >= 128 * 32 * 33 * 8 * 2
    assert L.cks_launch_count(g, L.CKS_BF16, L.CKS_OP_FWD) == 3
    g = L.make_geom(128, 3, 32, 32, 64, 3, 3, 1, 1, 1, 1)   # narrow row path: X read unpadded
    assert L.cks_workspace_size(g, L.CKS_BF16, L.CKS_OP_FWD) == 0
    assert L.cks_launch_count(g, L.CKS_BF16, L.CKS_OP_FWD) == 1
    assert L.cks_launch_count(g, L.CKS_TF32, L.CKS_OP_FWD) == 1   # TF32 filter-row kernel too
    gz = L.cks_choose_gz(g, L.CKS_BF16)
    # G_Z partials + KB-REDUCE, or the cluster reduce (neither): the launch count follows the workspace
    assert L.cks_launch_count(g, L.CKS_BF16, L.CKS_OP_WGRAD) == 1 + (L.cks_workspace_size(g, L.CKS_BF16, L.CKS_OP_WGRAD) > 0)
    g = L.make_geom(128, 64, 32, 32, 64, 3, 3, 2, 2, 1, 1)
    # W given: Stage1-free KS-deconv (one launch, no packed sub-filters in the
    # workspace) where the plan takes it, else KB-SPLIT + KB-KS
    direct = L.plan_dict(g, L.CKS_BF16, L.CKS_OP_DECONV)["ks_direct"] == "1"
    assert L.cks_launch_count(g, L.CKS_BF16, L.CKS_OP_DECONV) == (1 if direct else 2)
    assert L.cks_launch_count(g, L.CKS_BF16, L.CKS_OP_DECONV, c_packed_given=True) == 1
    g3 = L.make_geom(128, 3, 32, 32, 64, 3, 3, 2, 2, 1, 1)  # W rows of 6 bytes: not eligible
    assert L.plan_dict(g3, L.CKS_BF16, L.CKS_OP_DECONV)["ks_direct"] == "0"
    gz = L.cks_choose_gz(g, L.CKS_BF16)
    assert 1 <= gz <= 64
    # G_Z partials + KB-REDUCE, or the cluster reduce (neither): the launch count follows the workspace
    assert L.cks_launch_count(g, L.CKS_BF16, L.CKS_OP_WGRAD) == 1 + (L.cks_workspace_size(g, L.CKS_BF16, L.CKS_OP_WGRAD) > 0)
    # G_Z = 4 segments: either fp32 partials in the workspace + a KB-REDUCE launch,
    # or (one-wave grids, gz <= 8) the cluster reduce with neither
    ws = L.cks_workspace_size(g, L.CKS_BF16, L.CKS_OP_WGRAD, gz=4)
    n4 = L.cks_launch_count(g, L.CKS_BF16, L.CKS_OP_WGRAD, gz=4)
    assert (ws >= 4 * 64 * 9 * 64 * 4 and n4 == 2) or (ws == 0 and n4 == 1)
    g_big = L.make_geom(256, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1)   # 3 row tiles x gz 40: partials + reduce
    assert L.cks_workspace_size(g_big, L.CKS_BF16, L.CKS_OP_WGRAD, gz=40) >= 40 * 64 * 9 * 64 * 4
    assert L.cks_launch_count(g_big, L.CKS_BF16, L.CKS_OP_WGRAD, gz=40) == 2
    assert L.cks_ks_split_size(g, L.CKS_BF16) == 4 * 64 * 2 * 2 * 64 * 2


def _classes(desc: dict):
    return [tuple(int(v) for v in c.split(":")) for c in desc["cls"].split(",")]


def test_narrow_row_path_plan():
    """Narrow-channel layers take the filter-row kernels (kernels/narrow.cuh) in
    BF16 and TF32: no channel padding pass; the output columns are partitioned
    into classes (interior columns by box alignment, every border column its
    own class); the Sk-dilated G_Z is the total of the per-class segments
    (include/cks.h cks_choose_gz)."""
    for (C, W, FW, sw, OC) in [(3, 224, 7, 2, 64), (3, 32, 3, 1, 64), (3, 64, 4, 2, 128), (1, 16, 5, 1, 8),
                               (2, 24, 7, 3, 32), (4, 8, 3, 2, 8), (8, 16, 3, 1, 16), (16, 8, 3, 2, 40)]:
        g = L.make_geom(70, C, W, W, OC, FW, FW, sw, sw, FW // 2, FW // 2)
        OW = (W + 2 * (FW // 2) - FW) // sw + 1
        for dt in (L.CKS_BF16, L.CKS_TF32):
            eb = 2 if dt == L.CKS_BF16 else 4
            fwd, wg = L.plan_dict(g, dt, L.CKS_OP_FWD), L.plan_dict(g, dt, L.CKS_OP_WGRAD)
            if dt == L.CKS_TF32 and C > 8:
                assert fwd["kind"] == "igemm" and wg["kind"] == "wgrad", (C, W, FW, sw)
                continue
            assert fwd["kind"] == "row_fwd" and wg["kind"] == "row_wgrad", (C, W, FW, sw, dt)
            assert L.cks_launch_count(g, dt, L.CKS_OP_FWD) == 1          # no X/W padding pass
            for d in (fwd, wg):
                cls = _classes(d)
                cols = sorted(c0 + st * i for (c0, st, n, *_r) in cls for i in range(n))
                assert cols == list(range(OW)), (C, W, FW, sw, dt)    # classes partition the columns
                for (c0, st, n, off, kc0, kc1, base, cnt) in cls:
                    for i in range(n):
                        start = ((c0 + st * i) * sw - FW // 2) * C
                        assert ((start + off) * eb) % 16 == 0       # 16-byte aligned box origin
                        assert 0 <= kc0 < kc1 <= int(d["JB"]) * eb // 32
            gz = L.cks_choose_gz(g, dt)
            assert gz == int(wg["gz"]) and gz >= int(wg["classes"]), (C, W, FW, sw, gz)
            assert gz == sum(c[7] for c in _classes(wg))
            ocpad = OC % (8 if dt == L.CKS_BF16 else 4) != 0
            assert L.cks_launch_count(g, dt, L.CKS_OP_WGRAD) == 1 + ocpad + (gz > 1)
            ws = L.cks_workspace_size(g, dt, L.CKS_OP_WGRAD, gz=gz + 1)
            assert ws >= (gz + 1) * OC * FW * FW * C * 4
            # exact C-K-S at the K-chunk granularity: no ConvV2 product with a padding zero
            assert L.cks_padding_macs(g, dt, L.CKS_OP_FWD) == 0, (C, W, FW, sw, dt)
    # row pitch not a multiple of 16 bytes -> padded per-tap path
    g = L.make_geom(70, 3, 33, 33, 64, 3, 3, 1, 1, 1, 1)
    assert L.cks_launch_count(g, L.CKS_BF16, L.CKS_OP_FWD) == 3
    assert L.plan_dict(g, L.CKS_BF16, L.CKS_OP_FWD)["kind"] == "igemm"


def test_padding_macs_accounting():
    """cks_padding_macs: 0 for the trimmed-window kernels; the row-path Sk-dilated
    count equals a brute-force recount of the zero-filled operand rows inside its
    issued M-blocks (a stored dW row times a padding position of X)."""
    g = L.make_geom(256, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1)
    for op in (L.CKS_OP_FWD, L.CKS_OP_DECONV, L.CKS_OP_WGRAD):
        assert L.cks_padding_macs(g, L.CKS_BF16, op) == 0
    N, C, H, W, OC, F, s, p = 2, 3, 9, 8, 8, 3, 2, 1
    g = L.make_geom(N, C, H, W, OC, F, F, s, s, p, p)
    for dt in (L.CKS_BF16, L.CKS_TF32):
        d = L.plan_dict(g, dt, L.CKS_OP_WGRAD)
        assert d["kind"] == "row_wgrad"
        JB, R = int(d["JB"]), 128 // int(d["JB"])
        OH = (H + 2 * p - F) // s + 1
        n = 0
        for (c0, st, nc, off, *_r) in _classes(d):
            for i in range(nc):
                start = ((c0 + st * i) * s - p) * C
                for oh in range(OH):
                    ih0 = oh * s - p
                    fs, fe = max(-ih0, 0), min(H - ih0, F)
                    for m in range((F + R - 1) // R):
                        if not (m * R < fe and (m + 1) * R > fs):
                            continue
                        for fh in range(m * R, min((m + 1) * R, F)):
                            for e in range(JB):
                                j = off + e
                                if 0 <= j < F * C and (fh < fs or fh >= fe or not 0 <= start + j < W * C):
                                    n += 1
        assert L.cks_padding_macs(g, dt, L.CKS_OP_WGRAD) == n * OC * N


def test_zins_workspace_holds_the_zero_inserted_operand():
    """KB-ZINS workspace = staged operand with every structural zero of the
    textbook formulation (+ rotated filter + inner workspace): the sizes follow
    from P:114 / Table III's O_H^p = (O_H - 1)*sh + 1."""
    N, C, I, OC, F, s, p = 128, 64, 32, 128, 3, 2, 1
    g = L.make_geom(N, C, I, I, OC, F, F, s, s, p, p)
    O_ = (I + 2 * p - F) // s + 1                      # 16
    r = (I + 2 * p - F) % s                            # output padding (reading c10): 1
    q = F - 1 - p
    zd = (O_ - 1) * s + 1 + 2 * q + r                  # deconv staging extent: 34 = I + F - 1
    assert zd == I + F - 1
    assert L.cks_zins_workspace_size(g, L.CKS_BF16, L.CKS_OP_DECONV) >= N * zd * zd * OC * 2 + C * F * F * OC * 2
    zw = (O_ - 1) * s + 1 + r                          # wgrad: zero-inserted dY = unit-stride output extent
    assert zw == I + 2 * p - F + 1
    assert L.cks_zins_workspace_size(g, L.CKS_BF16, L.CKS_OP_WGRAD) >= N * zw * zw * OC * 2
    assert L.cks_zins_workspace_size(g, L.CKS_BF16, L.CKS_OP_FWD) >= N * (I + 2 * p) ** 2 * C * 2
    lib = L.lib()
    assert lib.cks_zins_deconv2d(ctypes.byref(g), 1, 16, 16, 16, None, 0, None) == 1     # ws required
    assert lib.cks_zins_wgrad(ctypes.byref(g), 1, 16, 16, 16, 16, 0, None) == 5          # ws too small
    bad = L.make_geom(1, 4, 8, 8, 8, 3, 3, 1, 1, 3, 1)
    with pytest.raises(L.CksError) as e:
        L.cks_zins_workspace_size(bad, L.CKS_BF16, L.CKS_OP_FWD)
    assert e.value.status == 2


def _plans(cfg, op, dt=None):
    """Tile plans the library picks for every layer of a config (cks_plan_describe, host only)."""
    from cks_synth import get_config
    dt = L.CKS_BF16 if dt is None else dt
    code = {"fwd": L.CKS_OP_FWD, "deconv": L.CKS_OP_DECONV, "wgrad": L.CKS_OP_WGRAD}[op]
    out = {}
    for lay in get_config(cfg)[1]:
        g = L.make_geom(lay.N, lay.C, lay.H, lay.W, lay.OC, lay.FH, lay.FW, lay.sh, lay.sw, lay.ph, lay.pw)
        out[lay.name] = L.plan_dict(g, dt, code)
    return out


def test_plan_choices_on_the_workloads():
    """Regression guard for the measured plan heuristics: CTA
    pairs on C3 l3 (one-pixel plans with >= 2 channel blocks, >= 2.5 waves),
    cluster split-K on the 4x4 C2 layers, single-CTA tiles elsewhere."""
    fwd3 = _plans(2, "fwd")
    assert fwd3["l3_0"]["pair"] == "1" and fwd3["l3a"]["pair"] == "1"
    assert fwd3["l4_0"]["pair"] == "0" and fwd3["l2_0"]["pair"] == "0"
    fwd2 = _plans(1, "fwd")
    assert fwd2["vgg4_512to512_s2"]["zc"] == "1" and int(fwd2["vgg4_512to512_s2"]["Z"]) >= 2
    assert fwd2["vgg32_64to64_s1"]["zc"] == "0" and fwd2["vgg32_64to64_s1"]["pair"] == "0"
    for name, pl in list(fwd2.items()) + list(fwd3.items()):
        if pl.get("zc") == "1":   # one wave of resident clusters
            assert int(pl["out_tiles"]) * int(pl["Z"]) <= 148, name


def test_mma_program_capacity_bound():
    """an igemm tile's MMA-program entries (<= pbw x taps per filter
    row) must fit the 64-entry lists; wide stride-2 filters narrow the pixel block."""
    for geo in [(128, 8, 128, 128, 32, 10, 10, 2, 2, 4, 4), (20, 8, 128, 128, 32, 10, 10, 2, 2, 4, 4),
                (128, 3, 224, 224, 64, 11, 11, 2, 2, 5, 5), (128, 3, 227, 227, 64, 11, 11, 4, 4, 0, 0),
                (64, 16, 64, 64, 32, 32, 32, 1, 1, 16, 16), (256, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1)]:
        g = L.make_geom(*geo)
        for dt in (L.CKS_BF16, L.CKS_TF32):
            for op in (L.CKS_OP_FWD, L.CKS_OP_DECONV):
                d = L.plan_dict(g, dt, op)
                if d["kind"] == "igemm":
                    assert int(d["pbw"]) * int(d["ntap"]) <= 64, (geo, dt, op, d)


def test_op_counts3_match_oracle():
    """3-D zero-free MAC counts: library (closed forms per axis) == oracle
    (enumeration of the valid (o, f) pairs), bit-exact."""
    from oracle import cks_oracle3d as O3
    rng = np.random.default_rng(12)
    n = 0
    while n < 200:
        f = [int(rng.integers(1, 6)) for _ in range(3)]
        s = [int(rng.integers(1, 5)) for _ in range(3)]
        p = [int(rng.integers(0, ff)) for ff in f]
        dhw = [int(rng.integers(1, 14)) for _ in range(3)]
        if any(i + 2 * pp - ff < 0 for i, ff, pp in zip(dhw, f, p)):
            continue
        N, C, OC = int(rng.integers(1, 5)), int(rng.integers(1, 9)), int(rng.integers(1, 9))
        g = L.make_geom3(N, C, *dhw, OC, *f, *s, *p)
        got = L.cks_op_counts3(g)
        ref = O3.op_counts3d(N, C, OC, dhw, f, s, p)
        assert got["zero_free_macs"] == ref["zero_free_macs"]
        assert [got["VD"], got["VH"], got["VW"]] == ref["V"]
        assert list(L.cks_output_shape3(g)) == ref["O"]
        n += 1


def test_row_group_plans():
    """Small per-GPU batches (N <= 64, e.g. C5 strong scaling: 256 / 8 = 32 images per GPU) tile M as
    128 / rg_ni output rows x rg_ni images (row groups) instead of 128 images of one pixel."""
    for N, want in [(1, 32), (20, 32), (32, 32), (33, 64), (64, 64), (65, 0), (128, 0), (256, 0)]:
        for geo in [(N, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1), (N, 128, 28, 28, 256, 3, 3, 2, 2, 1, 1),
                    (N, 64, 56, 56, 128, 1, 1, 2, 2, 0, 0)]:
            g = L.make_geom(*geo)
            for dt in (L.CKS_BF16, L.CKS_TF32):
                for op in (L.CKS_OP_FWD, L.CKS_OP_DECONV):
                    d = L.plan_dict(g, dt, op)
                    assert d["kind"] == "igemm" and int(d["rg"]) == want, (geo, dt, op, d)
                    if want:  # one activation column per A slot, no CTA pairs
                        assert d["apos"] == "1" and d["pair"] == "0", d


def test_row_group_wgrad_plans():
    """Sk-dilated at N <= kimg / 2: k-blocks of rg_pk output positions x rg images (position chunks)."""
    for N, rg in [(1, 16), (16, 16), (17, 32), (32, 32), (33, 0), (64, 0), (256, 0)]:
        for geo in [(N, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1), (N, 128, 28, 28, 256, 3, 3, 2, 2, 1, 1),
                    (N, 256, 14, 14, 256, 3, 3, 1, 1, 1, 1)]:
            for dt in (L.CKS_BF16, L.CKS_TF32):
                d = L.plan_dict(L.make_geom(*geo), dt, L.CKS_OP_WGRAD)
                assert d["kind"] == "wgrad", d
                want = rg if 2 * N <= int(d["kimg"]) else 0
                assert int(d["rg"]) == want, (geo, dt, d)
                if want:
                    assert int(d["rg_pk"]) * want == int(d["kimg"]) and d["pp"] == "0", d


def test_row_group_narrow_plans():
    """Narrow-channel (filter-row) kernels at small batches: ConvV2 row groups for N <= 64,
    Sk-dilated class-column k-blocks for N <= 32; batch-as-M / 64-image k-blocks above."""
    for N, want_f, want_w in [(1, 32, 16), (16, 32, 16), (32, 32, 32), (33, 64, 0), (64, 64, 0), (65, 0, 0),
                              (256, 0, 0)]:
        g = L.make_geom(N, 3, 224, 224, 64, 7, 7, 2, 2, 3, 3)
        for dt in (L.CKS_BF16, L.CKS_TF32):
            f = L.plan_dict(g, dt, L.CKS_OP_FWD)
            w = L.plan_dict(g, dt, L.CKS_OP_WGRAD)
            assert f["kind"] == "row_fwd" and int(f["rg"]) == want_f, (N, dt, f)
            assert w["kind"] == "row_wgrad" and int(w["rg"]) == want_w, (N, dt, w)
