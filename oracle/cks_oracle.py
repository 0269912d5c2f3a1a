"""fp64 CPU oracle for the C-K-S operators (arXiv 2306.15951).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product path (``paper_2306_15951_b200``) never imports it, and it
imports nothing from the product path: the two share no code.

Citations: ``P:<line>`` = /root/reference/PAPER.md line (section / equation /
algorithm).  Readings of garbled or ambiguous passages follow SURVEY.md §8(c)
(c1..c16) and are listed in DESIGN.md "Readings".

What is here
------------
1. The three operators as the paper DEFINES them, materialising every zero the
   paper talks about (the "common approach"):
     conv_ref    Eq (1) P:136 on the zero-padded X            (Fig. 1)
     deconv_ref  Eq (2): zero-inserted dY, padded, unit-stride
                 convolution with W^rot180
     wgrad_ref   Eq (3): zero-inserted dY used as the filter over the
                 zero-padded X ("dY serves as filters in dilated-convolution",
                 P:114; "dilate is equal to the stride")
   Each tap is one BLAS matmul over the channel axis (a library primitive used
   as a step); no blocking, fusion or zero skipping.
2. Row/element samplers of the same definitions, for full-size sampled parity.
3. Scalar brute force (pure Python loops) of the textbook index relation
   ``ih = oh*sh + fh - ph`` -- an independent formulation for tiny inputs.
4. The paper's algorithms step by step (Alg. 1, Alg. 2 Stage1/Stage2&3 +
   V2, Alg. 3 + 3B) with MAC counters, under readings c1-c6.  These
   reproduce the paper's printed complexity counts (Figs 4-8) and pin the
   readings against the definitions.
5. Integer tables T1-T4 by BRUTE-FORCE ENUMERATION of the valid pair set
   {(o, f): 0 <= o*s + f - p < I} per axis (never via closed forms), plus
   zero-free and nominal (Table III) operation counts.

Parity pins (tests/test_oracle.py): SPEC hand case, Fig. 4/5/6/7/8 + Table III
values on the worked-example geometry (reading c8), brute force, adjoint
identity, central finite differences, torch fp64 CPU conv routines, s=1 F=1
matmul special case, table partition invariants.  Nothing here is
"parity unpinned".
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# ---------------------------------------------------------------------------
# Geometry (Table I)
# ---------------------------------------------------------------------------


class GeometryError(ValueError):
    pass


@dataclass(frozen=True)
class Geom:
    """Table I symbols.  C = I_C, H/W = I_H/I_W (the X side)."""
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

    @property
    def OH(self):
        return out_extent(self.H, self.FH, self.sh, self.ph)

    @property
    def OW(self):
        return out_extent(self.W, self.FW, self.sw, self.pw)


def out_extent(I, F, s, p):
    """O = floor((I + 2p - F)/s) + 1 (Table I shape rule; reading c10)."""
    if s < 1 or p < 0 or F < 1 or I < 1:
        raise GeometryError("non-positive extent/stride or negative padding")
    if p >= F:
        # reading c16: every patch must intersect the valid region
        raise GeometryError("padding must be smaller than the filter")
    if I + 2 * p - F < 0:
        raise GeometryError("filter larger than padded input")
    return (I + 2 * p - F) // s + 1


def geom(**kw) -> Geom:
    g = Geom(**kw)
    g.OH, g.OW  # validate
    return g


# ---------------------------------------------------------------------------
# 1. The definitions (materialised zeros)
# ---------------------------------------------------------------------------


def zero_pad(X, ph, pw):
    """Zero-pad the two spatial axes of an NHWC tensor ("pad certain 0s
    on the boundary of input-feature-maps")."""
    N, H, W, C = X.shape
    Xp = np.zeros((N, H + 2 * ph, W + 2 * pw, C), dtype=np.float64)
    Xp[:, ph:ph + H, pw:pw + W, :] = X
    return Xp


def zero_insert(G, sh, sw):
    """Insert (stride-1) zeros between adjacent elements of dY.  The
    result has O_H^p = O_H + (O_H-1)(sh-1) rows (Table III)."""
    N, OH, OW, C = G.shape
    Z = np.zeros((N, (OH - 1) * sh + 1, (OW - 1) * sw + 1, C), dtype=np.float64)
    Z[:, ::sh, ::sw, :] = G
    return Z


def conv_ref(X, Wt, sh, sw, ph, pw):
    """Eq (1): Y[n,oh,ow,oc] = sum_{fh,fw,ic} Xpad[n, oh*sh+fh, ow*sw+fw, ic]
    * W[oc,fh,fw,ic] -- im2col view of Fig. 1, one matmul per tap."""
    X = np.asarray(X, dtype=np.float64)
    Wt = np.asarray(Wt, dtype=np.float64)
    N, H, Wd, C = X.shape
    OC, FH, FW, C2 = Wt.shape
    assert C == C2
    OH, OW = out_extent(H, FH, sh, ph), out_extent(Wd, FW, sw, pw)
    Xp = zero_pad(X, ph, pw)
    Y = np.zeros((N, OH, OW, OC), dtype=np.float64)
    for fh in range(FH):
        for fw in range(FW):
            patch = Xp[:, fh:fh + (OH - 1) * sh + 1:sh, fw:fw + (OW - 1) * sw + 1:sw, :]
            Y += patch @ Wt[:, fh, fw, :].T
    return Y


def rot180_swap(Wt):
    """W^rot180 of Eq (2) with the channel roles swapped for the deconvolution:
    R[ic, fh, fw, oc] = W[oc, F_H-1-fh, F_W-1-fw, ic]."""
    return np.ascontiguousarray(np.transpose(Wt[:, ::-1, ::-1, :], (3, 1, 2, 0)))


def deconv_ref(G, Wt, H, Wd, sh, sw, ph, pw):
    """Eq (2): dX = deconv2D(dY, W^rot180), the common approach: zero-
    insert dY, pad by q = F-1-p on the leading side and q + r on the
    trailing side, r = (I + 2p - F) mod s (output padding restoring the stored
    I; reading c10), then a unit-stride convolution with W^rot180."""
    G = np.asarray(G, dtype=np.float64)
    Wt = np.asarray(Wt, dtype=np.float64)
    OC, FH, FW, C = Wt.shape
    OH, OW = out_extent(H, FH, sh, ph), out_extent(Wd, FW, sw, pw)
    assert G.shape[1:] == (OH, OW, OC), (G.shape, (OH, OW, OC))
    Z = zero_insert(G, sh, sw)
    qh, qw = FH - 1 - ph, FW - 1 - pw
    rh, rw = (H + 2 * ph - FH) % sh, (Wd + 2 * pw - FW) % sw
    N = G.shape[0]
    Zp = np.zeros((N, Z.shape[1] + 2 * qh + rh, Z.shape[2] + 2 * qw + rw, OC))
    Zp[:, qh:qh + Z.shape[1], qw:qw + Z.shape[2], :] = Z
    R = rot180_swap(Wt)                      # [ic, fh, fw, oc]
    dX = conv_ref(Zp, R, 1, 1, 0, 0)
    assert dX.shape == (N, H, Wd, C), dX.shape
    return dX


def wgrad_ref(X, G, FH, FW, sh, sw, ph, pw):
    """Eq (3): dW = dilated_conv2D(X, dY): the zero-inserted dY acts as
    the filter (dilate = stride) over the zero-padded X:
    dW[oc,fh,fw,ic] = sum_{n,j,k} Xpad[n, j+fh, k+fw, ic] * Z[n,j,k,oc]."""
    X = np.asarray(X, dtype=np.float64)
    G = np.asarray(G, dtype=np.float64)
    N, H, Wd, C = X.shape
    OC = G.shape[3]
    OH, OW = out_extent(H, FH, sh, ph), out_extent(Wd, FW, sw, pw)
    assert G.shape == (N, OH, OW, OC)
    Xp = zero_pad(X, ph, pw)
    Z = zero_insert(G, sh, sw)
    OHp, OWp = Z.shape[1], Z.shape[2]
    dW = np.zeros((OC, FH, FW, C), dtype=np.float64)
    Zf = Z.reshape(-1, OC)
    for fh in range(FH):
        for fw in range(FW):
            dW[:, fh, fw, :] = Zf.T @ Xp[:, fh:fh + OHp, fw:fw + OWp, :].reshape(-1, C)
    return dW


# ---------------------------------------------------------------------------
# 2. Samplers of the same definitions (full-size parity on sampled outputs)
# ---------------------------------------------------------------------------


def conv_ref_rows(X, Wt, sh, sw, ph, pw, samples):
    """Y[n, oh, ow, :] for each (n, oh, ow) in ``samples`` by Eq (1) on the
    zero-padded image n (same definition as conv_ref, one patch at a time)."""
    OC, FH, FW, C = Wt.shape
    Wf = np.asarray(Wt, dtype=np.float64).reshape(OC, -1)
    out = np.zeros((len(samples), OC))
    cache = {}
    for i, (n, oh, ow) in enumerate(samples):
        if n not in cache:
            cache = {n: zero_pad(np.asarray(X[n:n + 1], dtype=np.float64), ph, pw)[0]}
        Xp = cache[n]
        patch = Xp[oh * sh:oh * sh + FH, ow * sw:ow * sw + FW, :]
        out[i] = Wf @ patch.reshape(-1)
    return out


def deconv_ref_rows(G, Wt, H, Wd, sh, sw, ph, pw, samples):
    """dX[n, ih, iw, :] for each sample by Eq (2) (zero-inserted, padded dY of
    image n convolved with W^rot180 at one position)."""
    OC, FH, FW, C = Wt.shape
    R = rot180_swap(np.asarray(Wt, dtype=np.float64)).reshape(C, -1)
    qh, qw = FH - 1 - ph, FW - 1 - pw
    rh, rw = (H + 2 * ph - FH) % sh, (Wd + 2 * pw - FW) % sw
    out = np.zeros((len(samples), C))
    cache = {}
    for i, (n, ih, iw) in enumerate(samples):
        if n not in cache:
            Z = zero_insert(np.asarray(G[n:n + 1], dtype=np.float64), sh, sw)[0]
            Zp = np.zeros((Z.shape[0] + 2 * qh + rh, Z.shape[1] + 2 * qw + rw, OC))
            Zp[qh:qh + Z.shape[0], qw:qw + Z.shape[1], :] = Z
            cache = {n: Zp}
        Zp = cache[n]
        out[i] = R @ Zp[ih:ih + FH, iw:iw + FW, :].reshape(-1)
    return out


def wgrad_ref_taps(X, G, FH, FW, sh, sw, ph, pw, taps, n_chunk=16):
    """dW[:, fh, fw, :] for each (fh, fw) in ``taps`` by Eq (3), accumulated
    image chunk by image chunk (same sum as wgrad_ref, bounded memory)."""
    N, H, Wd, C = X.shape
    OC = G.shape[3]
    out = np.zeros((len(taps), OC, C))
    for n0 in range(0, N, n_chunk):
        Xp = zero_pad(np.asarray(X[n0:n0 + n_chunk], dtype=np.float64), ph, pw)
        Z = zero_insert(np.asarray(G[n0:n0 + n_chunk], dtype=np.float64), sh, sw)
        OHp, OWp = Z.shape[1], Z.shape[2]
        Zf = Z.reshape(-1, OC)
        for t, (fh, fw) in enumerate(taps):
            out[t] += Zf.T @ Xp[:, fh:fh + OHp, fw:fw + OWp, :].reshape(-1, C)
    return out


# ---------------------------------------------------------------------------
# 3. Scalar brute force (tiny inputs only)
# ---------------------------------------------------------------------------


def brute_conv(X, Wt, sh, sw, ph, pw):
    """Textbook loop: Y[n,oh,ow,oc] += X[n,ih,iw,ic]*W[oc,fh,fw,ic] for every
    in-range ih = oh*sh+fh-ph, iw = ow*sw+fw-pw."""
    N, H, Wd, C = X.shape
    OC, FH, FW, _ = Wt.shape
    OH, OW = out_extent(H, FH, sh, ph), out_extent(Wd, FW, sw, pw)
    Y = np.zeros((N, OH, OW, OC))
    for n in range(N):
        for oh in range(OH):
            for ow in range(OW):
                for oc in range(OC):
                    acc = 0.0
                    for fh in range(FH):
                        ih = oh * sh + fh - ph
                        if not 0 <= ih < H:
                            continue
                        for fw in range(FW):
                            iw = ow * sw + fw - pw
                            if not 0 <= iw < Wd:
                                continue
                            for ic in range(C):
                                acc += float(X[n, ih, iw, ic]) * float(Wt[oc, fh, fw, ic])
                    Y[n, oh, ow, oc] = acc
    return Y


def brute_deconv(G, Wt, H, Wd, sh, sw, ph, pw):
    """Scatter form of the adjoint of brute_conv (chain rule of Eq (1))."""
    N, OH, OW, OC = G.shape
    _, FH, FW, C = Wt.shape
    dX = np.zeros((N, H, Wd, C))
    for n in range(N):
        for oh in range(OH):
            for ow in range(OW):
                for fh in range(FH):
                    ih = oh * sh + fh - ph
                    if not 0 <= ih < H:
                        continue
                    for fw in range(FW):
                        iw = ow * sw + fw - pw
                        if not 0 <= iw < Wd:
                            continue
                        for oc in range(OC):
                            g = float(G[n, oh, ow, oc])
                            for ic in range(C):
                                dX[n, ih, iw, ic] += g * float(Wt[oc, fh, fw, ic])
    return dX


def brute_wgrad(X, G, FH, FW, sh, sw, ph, pw):
    N, H, Wd, C = X.shape
    _, OH, OW, OC = G.shape
    dW = np.zeros((OC, FH, FW, C))
    for oc in range(OC):
        for fh in range(FH):
            for fw in range(FW):
                for ic in range(C):
                    acc = 0.0
                    for n in range(N):
                        for oh in range(OH):
                            ih = oh * sh + fh - ph
                            if not 0 <= ih < H:
                                continue
                            for ow in range(OW):
                                iw = ow * sw + fw - pw
                                if not 0 <= iw < Wd:
                                    continue
                                acc += float(X[n, ih, iw, ic]) * float(G[n, oh, ow, oc])
                    dW[oc, fh, fw, ic] = acc
    return dW


# ---------------------------------------------------------------------------
# 4. The paper's algorithms, step by step (Appendix)
# ---------------------------------------------------------------------------


def ceil_div(a, b):
    """Mathematical ceiling (correct for negative a; SURVEY.md §8 notation)."""
    return -((-a) // b)


def convv2_alg(X, Wt, sh, sw, ph, pw, trim=True):
    """Alg. 1 ConvV2 with reading c1 (half-open [fh_s, fh_e)):
    (ih_s, iw_s) = (oh, ow) (.) (sh, sw) - (ph, pw);
    fh_s = max(-ih_s, 0), fh_e = min(I_H - ih_s, F_H)  (same on w);
    Y = sum_{fh in [fh_s,fh_e), fw in [fw_s,fw_e), ic} X[n, ih_s+fh, iw_s+fw, ic] W[oc,fh,fw,ic].
    trim=False is "normal convolution" over the whole padded patch (Fig. 1);
    returns (Y, MACs) with MACs counted per (n, oh, ow, oc) dot-product term
    over channels (the paper's counts use I_C = O_C = N = 1)."""
    X = np.asarray(X, dtype=np.float64)
    Wt = np.asarray(Wt, dtype=np.float64)
    N, H, Wd, C = X.shape
    OC, FH, FW, _ = Wt.shape
    OH, OW = out_extent(H, FH, sh, ph), out_extent(Wd, FW, sw, pw)
    Xp = zero_pad(X, ph, pw)
    Y = np.zeros((N, OH, OW, OC))
    macs = 0
    for oh in range(OH):
        for ow in range(OW):
            ih_s, iw_s = oh * sh - ph, ow * sw - pw
            if trim:
                fh_s, fh_e = max(-ih_s, 0), min(H - ih_s, FH)
                fw_s, fw_e = max(-iw_s, 0), min(Wd - iw_s, FW)
            else:
                fh_s, fh_e, fw_s, fw_e = 0, FH, 0, FW
            # patch of the padded X = X[ih_s+fh] for in-range rows
            patch = Xp[:, ih_s + ph + fh_s:ih_s + ph + fh_e, iw_s + pw + fw_s:iw_s + pw + fw_e, :]
            Wsub = Wt[:, fh_s:fh_e, fw_s:fw_e, :]
            Y[:, oh, ow, :] = patch.reshape(N, -1) @ Wsub.reshape(OC, -1).T
            macs += N * OC * C * (fh_e - fh_s) * (fw_e - fw_s)
    return Y, macs


def ks_split_alg(Wt, sh, sw):
    """Alg. 2 Stage1 (Fig. 5): rotate W by 180 degrees and split
    into sh*sw smaller kernels.  Reading c2: C is
    sh x sw x O_C x ceil(F_H/sh) x ceil(F_W/sw) x I_C (zero-initialised);
    <oph, opw>_{y,x} = <ceil((F_H-y)/sh), ceil((F_W-x)/sw)> - 1;
    <fh, fw> = <y, x> + <oph - ch, opw - cw> (.) <sh, sw>;
    C[y,x,oc,ch,cw,:] = W[oc,fh,fw,:] if <fh,fw> in-range-of W.
    Returns (C, CH[y], CW[x]) where C_{y,x} has spatial extent CH[y] x CW[x]."""
    Wt = np.asarray(Wt, dtype=np.float64)
    OC, FH, FW, C = Wt.shape
    CHm, CWm = ceil_div(FH, sh), ceil_div(FW, sw)
    Cker = np.zeros((sh, sw, OC, CHm, CWm, C))
    CH = [ceil_div(FH - y, sh) for y in range(sh)]
    CW = [ceil_div(FW - x, sw) for x in range(sw)]
    for y in range(sh):
        for x in range(sw):
            oph, opw = CH[y] - 1, CW[x] - 1
            for ch in range(CHm):
                for cw in range(CWm):
                    fh = y + (oph - ch) * sh
                    fw = x + (opw - cw) * sw
                    if 0 <= fh < FH and 0 <= fw < FW:
                        Cker[y, x, :, ch, cw, :] = Wt[:, fh, fw, :]
    return Cker, CH, CW


def ks_deconv_alg(G, Cker, CH, CW, H, Wd, sh, sw, ph, pw, trim=True):
    """Alg. 2 Stage2&3 and, with trim=True, Alg. 2B KS-deconv-V2.
    Readings: c3 -- rows u range over all u with ih = u*sh + ih_s < I_H;
    c4 -- the V2 trim end is min(O_H - oh_s, CH_y); c11 -- dX = 0 first.
    Per phase (y, x):
      <ih_s, iw_s> = <y, x> - <ph, pw>, then += ceil(-ih_s/sh)*sh if negative;
      <oh_s, ow_s> = <(ih+ph-y)/sh, (iw+pw-x)/sw> - <oph, opw>   (exact)
      dX[n,ih,iw,ic] += dY[n, oh_s+ch, ow_s+cw, oc] * C[y,x,oc,ch,cw,ic]
    for (oh, ow) in-range-of dY.  Returns (dX, MACs) counted like convv2_alg
    (Stage2 MACs; Fig. 5 "72", Fig. 6 "50")."""
    G = np.asarray(G, dtype=np.float64)
    N, OH, OW, OC = G.shape
    C = Cker.shape[-1]
    dX = np.zeros((N, H, Wd, C))              # Alg. 2: dX initialised to 0
    macs = 0
    for y in range(sh):
        for x in range(sw):
            oph, opw = CH[y] - 1, CW[x] - 1
            ih_s, iw_s = y - ph, x - pw
            if ih_s < 0:
                ih_s += ceil_div(-ih_s, sh) * sh
            if iw_s < 0:
                iw_s += ceil_div(-iw_s, sw) * sw
            if CH[y] == 0 or CW[x] == 0:
                continue                      # empty phase: dX stays 0 (c11)
            u = 0
            while u * sh + ih_s < H:
                ih = u * sh + ih_s
                assert (ih + ph - y) % sh == 0
                oh_s = (ih + ph - y) // sh - oph
                if trim:
                    ch_s, ch_e = max(-oh_s, 0), min(OH - oh_s, CH[y])
                else:
                    ch_s, ch_e = 0, CH[y]
                v = 0
                while v * sw + iw_s < Wd:
                    iw = v * sw + iw_s
                    ow_s = (iw + pw - x) // sw - opw
                    if trim:
                        cw_s, cw_e = max(-ow_s, 0), min(OW - ow_s, CW[x])
                    else:
                        cw_s, cw_e = 0, CW[x]
                    acc = np.zeros((N, C))
                    for ch in range(ch_s, ch_e):
                        oh = oh_s + ch
                        for cw in range(cw_s, cw_e):
                            ow = ow_s + cw
                            macs += N * OC * C
                            if not (0 <= oh < OH and 0 <= ow < OW):
                                continue      # V1 multiplies a (padded) zero here
                            acc += G[:, oh, ow, :] @ Cker[y, x, :, ch, cw, :]
                    dX[:, ih, iw, :] = acc
                    v += 1
                u += 1
    return dX, macs


def sk_dilated_alg(X, G, FH, FW, sh, sw, ph, pw, trim=True, visit=None):
    """Alg. 3 Sk-dilated and, with trim=True, Alg. 3B Sk-dilated-V2.
    Leaping access: the filter dY is read with unit step, X with
    step = stride.  Readings: c5 -- oh_s = max(ceil(-ih_s/sh), 0),
    oh_e = min(O_H, ceil((I_H - ih_s)/sh)) with ih_s = fh - ph; c6 -- the
    range check is on X.  ``visit`` (optional list) records the X (ih, iw)
    sequence of the first (fh, fw, n, ic, oc) dot product (Fig. 7).
    Returns (dW, MACs)."""
    X = np.asarray(X, dtype=np.float64)
    G = np.asarray(G, dtype=np.float64)
    N, H, Wd, C = X.shape
    _, OH, OW, OC = G.shape
    dW = np.zeros((OC, FH, FW, C))
    macs = 0
    for fh in range(FH):
        for fw in range(FW):
            ih_s, iw_s = fh - ph, fw - pw
            if trim:
                oh_s, oh_e = max(ceil_div(-ih_s, sh), 0), min(OH, ceil_div(H - ih_s, sh))
                ow_s, ow_e = max(ceil_div(-iw_s, sw), 0), min(OW, ceil_div(Wd - iw_s, sw))
            else:
                oh_s, oh_e, ow_s, ow_e = 0, OH, 0, OW
            acc = np.zeros((OC, C))
            for oh in range(oh_s, oh_e):
                ih = ih_s + oh * sh
                for ow in range(ow_s, ow_e):
                    iw = iw_s + ow * sw
                    macs += N * OC * C
                    if visit is not None and (fh, fw) == visit[0]:
                        visit[1].append((ih, iw))
                    if not (0 <= ih < H and 0 <= iw < Wd):
                        continue              # V1 multiplies a padded zero here
                    acc += G[:, oh, ow, :].T @ X[:, ih, iw, :]
            dW[:, fh, fw, :] = acc
    return dW, macs


# ---------------------------------------------------------------------------
# 5. Integer tables by brute-force enumeration
# ---------------------------------------------------------------------------


def valid_pairs(I, F, s, p):
    """{(o, f): 0 <= o*s + f - p < I, 0 <= o < O, 0 <= f < F} by enumeration."""
    O = out_extent(I, F, s, p)
    return O, [(o, f) for o in range(O) for f in range(F) if 0 <= o * s + f - p < I]


def table_T1(I, F, s, p):
    """ConvV2 trim per output index: rows (o, ih_s = o*s - p, f_s, f_e) with
    [f_s, f_e) the valid f for o (Alg. 1, Fig. 4)."""
    O, pairs = valid_pairs(I, F, s, p)
    rows = []
    for o in range(O):
        fs = [f for (oo, f) in pairs if oo == o]
        assert fs and fs == list(range(fs[0], fs[-1] + 1)), "valid f not an interval"
        rows.append((o, o * s - p, fs[0], fs[-1] + 1))
    return rows


def table_T3(I, F, s, p):
    """Sk-dilated-V2 per tap f: (f, ih_s = f - p, oh_s, oh_e), [oh_s, oh_e) the
    valid o for f (Alg. 3B, Fig. 8).  Empty ranges give oh_s = oh_e = 0."""
    O, pairs = valid_pairs(I, F, s, p)
    rows = []
    for f in range(F):
        os_ = [o for (o, ff) in pairs if ff == f]
        if os_:
            assert os_ == list(range(os_[0], os_[-1] + 1))
            rows.append((f, f - p, os_[0], os_[-1] + 1))
        else:
            rows.append((f, f - p, 0, 0))
    return rows


def table_T2(I, F, s, p):
    """KS phases (Alg. 2, Fig. 5).  Brute force over the index
    relation o*s + f - p = i:
      phase y owns the taps f = y + j*s (j >= 0), CH_y = their count,
      oph_y = CH_y - 1, sub-filter tap ch <-> j = oph_y - ch (rot180);
      ih_s = the smallest i >= 0 with (i + p - y) divisible by s;
      rows i = u*s + ih_s < I, U_y = their count;
      per row: oh(ch) = (i + p - f(ch))/s, oh_s = oh(0), and [ch_s, ch_e)
      = {ch : 0 <= oh(ch) < O}; a_y = oh_s(u=0) (so oh(ch) = u + a_y + ch).
    Returns list of phase dicts."""
    O = out_extent(I, F, s, p)
    phases = []
    for y in range(s):
        taps = [f for f in range(F) if f % s == y]
        CH = len(taps)
        oph = CH - 1
        ih_s = next(i for i in range(s) if (i + p - y) % s == 0)
        rows = []
        u = 0
        while u * s + ih_s < I:
            i = u * s + ih_s
            if CH == 0:                       # empty phase (c11): convention
                rows.append((u, i, 0, 0, 0))  # oh_s = ch_s = ch_e = 0
                u += 1
                continue
            f0 = y + oph * s                  # tap of ch = 0
            oh_s = (i + p - f0) // s
            assert (i + p - f0) % s == 0
            chs = [ch for ch in range(CH)
                   if 0 <= (i + p - (y + (oph - ch) * s)) // s < O]
            if chs:
                assert chs == list(range(chs[0], chs[-1] + 1))
                ch_s, ch_e = chs[0], chs[-1] + 1
            else:
                ch_s = ch_e = 0
            rows.append((u, i, oh_s, ch_s, ch_e))
            u += 1
        a = rows[0][2] if rows else 0
        phases.append(dict(y=y, CH=CH, oph=oph, ih_s=ih_s, U=len(rows), a=a, rows=rows))
    return phases


def table_T4(I, F, s, p):
    """Trim classes: maximal runs of consecutive o with equal (f_s, f_e):
    rows (o_start, o_end, f_s, f_e).  The 2-D regions are their products."""
    rows = table_T1(I, F, s, p)
    runs = []
    for (o, _, fs, fe) in rows:
        if runs and runs[-1][2] == fs and runs[-1][3] == fe and runs[-1][1] == o:
            runs[-1][1] = o + 1
        else:
            runs.append([o, o + 1, fs, fe])
    return [tuple(r) for r in runs]


def axis_V(I, F, s, p):
    """Number of valid (o, f) pairs on one axis."""
    return len(valid_pairs(I, F, s, p)[1])


def op_counts(g: Geom):
    """Zero-free MACs (identical for all three operators)
    and the Table III nominal counts as FLOPs.  T_Dilated carries
    the N factor (reading c9) and is also returned without it."""
    VH = axis_V(g.H, g.FH, g.sh, g.ph)
    VW = axis_V(g.W, g.FW, g.sw, g.pw)
    OH, OW = g.OH, g.OW
    OHp = OH + (OH - 1) * (g.sh - 1)
    OWp = OW + (OW - 1) * (g.sw - 1)
    return dict(
        zero_free_macs=g.N * g.C * g.OC * VH * VW,
        zero_free_flops=2 * g.N * g.C * g.OC * VH * VW,
        T_conv=2 * (g.OC * g.N * OH * OW * g.FH * g.FW * g.C),
        T_deconv=2 * (g.C * g.N * g.H * g.W * g.FH * g.FW * g.OC),
        T_dilated=2 * (g.OC * g.FH * g.FW * g.C * OHp * OWp) * g.N,
        T_dilated_noN=2 * (g.OC * g.FH * g.FW * g.C * OHp * OWp),
        VH=VH, VW=VW, OHp=OHp, OWp=OWp,
    )


__all__ = [n for n in dir() if not n.startswith("_") and n not in ("annotations", "math", "np", "dataclass")]
