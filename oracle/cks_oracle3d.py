"""fp64 CPU oracle for the 3-D C-K-S operators.

TEST INFRASTRUCTURE ONLY (same rules as oracle/cks_oracle.py: imported by
``tests/`` only; shares no code with the product path).

The paper states the operators in 2-D and generalises them: "KS-deconv and
Sk-dilated convert sparse tensors to dense tensors, enabling stride^N and
dilate^N times acceleration for N-dimensional deconvolution and dilated-
convolution" (§I) and "The higher-dimensional versions of the C-K-S can
be analogized to its 2D counterpart" (§VI).  Reading c17:
the 3-D operators are Eqs (1)-(3) with a third spatial axis (depth D, filter
F_D, stride s_d, padding p_d) treated exactly like H and W -- zero padding on
every axis (Fig. 1), (s-1) zeros inserted between elements along every
axis, output extents by the Table I rule per axis.

Layouts: X [N][D][H][W][C], W [OC][FD][FH][FW][C], Y / dY [N][OD][OH][OW][OC].
Each definition materialises every zero and does one BLAS matmul per tap.
"""
from __future__ import annotations

import numpy as np

from .cks_oracle import out_extent


def zero_pad3(X, pd, ph, pw):
    """Zero-pad the three spatial axes of an NDHWC tensor."""
    N, D, H, W, C = X.shape
    Xp = np.zeros((N, D + 2 * pd, H + 2 * ph, W + 2 * pw, C), dtype=np.float64)
    Xp[:, pd:pd + D, ph:ph + H, pw:pw + W, :] = X
    return Xp


def zero_insert3(G, sd, sh, sw):
    """(s-1) zeros between adjacent elements along each spatial axis."""
    N, OD, OH, OW, C = G.shape
    Z = np.zeros((N, (OD - 1) * sd + 1, (OH - 1) * sh + 1, (OW - 1) * sw + 1, C), dtype=np.float64)
    Z[:, ::sd, ::sh, ::sw, :] = G
    return Z


def conv3d_ref(X, Wt, s, p):
    """Eq (1) in 3-D: Y[n,od,oh,ow,oc] = sum_{fd,fh,fw,ic}
    Xpad[n, od*sd+fd, oh*sh+fh, ow*sw+fw, ic] * W[oc,fd,fh,fw,ic]."""
    X = np.asarray(X, dtype=np.float64)
    Wt = np.asarray(Wt, dtype=np.float64)
    (sd, sh, sw), (pd, ph, pw) = s, p
    N, D, H, Wd, C = X.shape
    OC, FD, FH, FW, C2 = Wt.shape
    assert C == C2
    OD, OH, OW = out_extent(D, FD, sd, pd), out_extent(H, FH, sh, ph), out_extent(Wd, FW, sw, pw)
    Xp = zero_pad3(X, pd, ph, pw)
    Y = np.zeros((N, OD, OH, OW, OC), dtype=np.float64)
    for fd in range(FD):
        for fh in range(FH):
            for fw in range(FW):
                patch = Xp[:, fd:fd + (OD - 1) * sd + 1:sd, fh:fh + (OH - 1) * sh + 1:sh,
                           fw:fw + (OW - 1) * sw + 1:sw, :]
                Y += patch @ Wt[:, fd, fh, fw, :].T
    return Y


def rot180_swap3(Wt):
    """W rotated by 180 degrees on all three spatial axes, channels swapped:
    R[ic, fd, fh, fw, oc] = W[oc, FD-1-fd, FH-1-fh, FW-1-fw, ic]."""
    return np.ascontiguousarray(np.transpose(Wt[:, ::-1, ::-1, ::-1, :], (4, 1, 2, 3, 0)))


def deconv3d_ref(G, Wt, in_dhw, s, p):
    """Eq (2) in 3-D, the common approach: zero-insert dY along every axis,
    pad by q = F-1-p before and q + r after (r = (I+2p-F) mod s, reading c10),
    unit-stride convolution with W^rot180 (channels swapped)."""
    G = np.asarray(G, dtype=np.float64)
    Wt = np.asarray(Wt, dtype=np.float64)
    (D, H, Wd), (sd, sh, sw), (pd, ph, pw) = in_dhw, s, p
    OC, FD, FH, FW, C = Wt.shape
    OD, OH, OW = out_extent(D, FD, sd, pd), out_extent(H, FH, sh, ph), out_extent(Wd, FW, sw, pw)
    assert G.shape[1:] == (OD, OH, OW, OC), (G.shape, (OD, OH, OW, OC))
    Z = zero_insert3(G, sd, sh, sw)
    q = (FD - 1 - pd, FH - 1 - ph, FW - 1 - pw)
    r = ((D + 2 * pd - FD) % sd, (H + 2 * ph - FH) % sh, (Wd + 2 * pw - FW) % sw)
    N = G.shape[0]
    Zp = np.zeros((N, Z.shape[1] + 2 * q[0] + r[0], Z.shape[2] + 2 * q[1] + r[1], Z.shape[3] + 2 * q[2] + r[2], OC))
    Zp[:, q[0]:q[0] + Z.shape[1], q[1]:q[1] + Z.shape[2], q[2]:q[2] + Z.shape[3], :] = Z
    dX = conv3d_ref(Zp, rot180_swap3(Wt), (1, 1, 1), (0, 0, 0))
    assert dX.shape == (N, D, H, Wd, C), dX.shape
    return dX


def wgrad3d_ref(X, G, f, s, p):
    """Eq (3) in 3-D: the zero-inserted dY is the filter (dilate = stride,
    P:206) over the zero-padded X:
    dW[oc,fd,fh,fw,ic] = sum_{n,i,j,k} Xpad[n, i+fd, j+fh, k+fw, ic] * Z[n,i,j,k,oc]."""
    X = np.asarray(X, dtype=np.float64)
    G = np.asarray(G, dtype=np.float64)
    (FD, FH, FW), (sd, sh, sw), (pd, ph, pw) = f, s, p
    N, D, H, Wd, C = X.shape
    OC = G.shape[4]
    Xp = zero_pad3(X, pd, ph, pw)
    Z = zero_insert3(G, sd, sh, sw)
    ODp, OHp, OWp = Z.shape[1:4]
    Zf = Z.reshape(-1, OC)
    dW = np.zeros((OC, FD, FH, FW, C), dtype=np.float64)
    for fd in range(FD):
        for fh in range(FH):
            for fw in range(FW):
                dW[:, fd, fh, fw, :] = Zf.T @ Xp[:, fd:fd + ODp, fh:fh + OHp, fw:fw + OWp, :].reshape(-1, C)
    return dW


# ------------------------------------------------ scalar brute force (tiny inputs)
def brute_conv3d(X, Wt, s, p):
    """Textbook index relation i = o*s + f - p on every axis, scalar loops."""
    (sd, sh, sw), (pd, ph, pw) = s, p
    N, D, H, Wd, C = X.shape
    OC, FD, FH, FW, _ = Wt.shape
    OD, OH, OW = out_extent(D, FD, sd, pd), out_extent(H, FH, sh, ph), out_extent(Wd, FW, sw, pw)
    Y = np.zeros((N, OD, OH, OW, OC))
    for n in range(N):
        for od in range(OD):
            for oh in range(OH):
                for ow in range(OW):
                    for oc in range(OC):
                        acc = 0.0
                        for fd in range(FD):
                            i_d = od * sd + fd - pd
                            if not 0 <= i_d < D:
                                continue
                            for fh in range(FH):
                                ih = oh * sh + fh - ph
                                if not 0 <= ih < H:
                                    continue
                                for fw in range(FW):
                                    iw = ow * sw + fw - pw
                                    if 0 <= iw < Wd:
                                        acc += float(np.dot(X[n, i_d, ih, iw, :], Wt[oc, fd, fh, fw, :]))
                        Y[n, od, oh, ow, oc] = acc
    return Y


def brute_deconv3d(G, Wt, in_dhw, s, p):
    """dX[n,i,c] = sum over (o, f) with i = o*s + f - p of dY[n,o,oc] * W[oc,f,c]."""
    (D, H, Wd), (sd, sh, sw), (pd, ph, pw) = in_dhw, s, p
    N, OD, OH, OW, OC = G.shape
    _, FD, FH, FW, C = Wt.shape
    dX = np.zeros((N, D, H, Wd, C))
    for n in range(N):
        for od in range(OD):
            for oh in range(OH):
                for ow in range(OW):
                    for fd in range(FD):
                        i_d = od * sd + fd - pd
                        if not 0 <= i_d < D:
                            continue
                        for fh in range(FH):
                            ih = oh * sh + fh - ph
                            if not 0 <= ih < H:
                                continue
                            for fw in range(FW):
                                iw = ow * sw + fw - pw
                                if 0 <= iw < Wd:
                                    dX[n, i_d, ih, iw, :] += G[n, od, oh, ow, :] @ Wt[:, fd, fh, fw, :]
    return dX


def brute_wgrad3d(X, G, f, s, p):
    """dW[oc,f,c] = sum over n and o with i = o*s + f - p valid of X[n,i,c] * dY[n,o,oc]."""
    (FD, FH, FW), (sd, sh, sw), (pd, ph, pw) = f, s, p
    N, D, H, Wd, C = X.shape
    _, OD, OH, OW, OC = G.shape
    dW = np.zeros((OC, FD, FH, FW, C))
    for n in range(N):
        for od in range(OD):
            for oh in range(OH):
                for ow in range(OW):
                    for fd in range(FD):
                        i_d = od * sd + fd - pd
                        if not 0 <= i_d < D:
                            continue
                        for fh in range(FH):
                            ih = oh * sh + fh - ph
                            if not 0 <= ih < H:
                                continue
                            for fw in range(FW):
                                iw = ow * sw + fw - pw
                                if 0 <= iw < Wd:
                                    dW[:, fd, fh, fw, :] += np.outer(G[n, od, oh, ow, :], X[n, i_d, ih, iw, :])
    return dW


# ------------------------------------------------ sampled outputs (full-size parity)
def conv3d_ref_rows(X, Wt, s, p, samples):
    """Y[n, od, oh, ow, :] for each sample by Eq (1) on the zero-padded image n."""
    (sd, sh, sw), (pd, ph, pw) = s, p
    OC, FD, FH, FW, C = Wt.shape
    Wf = np.asarray(Wt, dtype=np.float64).reshape(OC, -1)
    out = np.zeros((len(samples), OC))
    for k, (n, od, oh, ow) in enumerate(samples):
        Xp = zero_pad3(np.asarray(X[n:n + 1], dtype=np.float64), pd, ph, pw)[0]
        patch = Xp[od * sd:od * sd + FD, oh * sh:oh * sh + FH, ow * sw:ow * sw + FW, :]
        out[k] = Wf @ patch.reshape(-1)
    return out


def wgrad3d_ref_taps(X, G, f, s, p, taps):
    """dW[:, fd, fh, fw, :] for each tap of ``taps`` by Eq (3)."""
    (FD, FH, FW), (sd, sh, sw), (pd, ph, pw) = f, s, p
    N, D, H, Wd, C = X.shape
    OC = G.shape[4]
    out = np.zeros((len(taps), OC, C))
    Xp = zero_pad3(np.asarray(X, dtype=np.float64), pd, ph, pw)
    Z = zero_insert3(np.asarray(G, dtype=np.float64), sd, sh, sw)
    ODp, OHp, OWp = Z.shape[1:4]
    Zf = Z.reshape(-1, OC)
    for k, (fd, fh, fw) in enumerate(taps):
        out[k] = Zf.T @ Xp[:, fd:fd + ODp, fh:fh + OHp, fw:fw + OWp, :].reshape(-1, C)
    return out


# ------------------------------------------------ counts
def valid_pairs_count(I, F, s, p):
    """#{(o, f): 0 <= o*s + f - p < I} by enumeration (one axis)."""
    O = out_extent(I, F, s, p)
    return sum(1 for o in range(O) for f in range(F) if 0 <= o * s + f - p < I)


def op_counts3d(N, C, OC, dhw, f, s, p):
    """Zero-free MACs N*C*OC*V_D*V_H*V_W (every 3-D C-K-S operator) and the
    nominal counts of the zero-materialising formulation (Table III, P:278-285,
    with the third axis): conv over padded X, deconv over the zero-inserted,
    padded dY, dilated over the zero-inserted dY as filter (N included, c9)."""
    V = [valid_pairs_count(I, F, ss, pp) for I, F, ss, pp in zip(dhw, f, s, p)]
    O = [out_extent(I, F, ss, pp) for I, F, ss, pp in zip(dhw, f, s, p)]
    Op = [(o - 1) * ss + 1 for o, ss in zip(O, s)]
    taps = f[0] * f[1] * f[2]
    return dict(zero_free_macs=N * C * OC * V[0] * V[1] * V[2],
                nominal_macs_conv=N * OC * O[0] * O[1] * O[2] * taps * C,
                nominal_macs_deconv=N * C * dhw[0] * dhw[1] * dhw[2] * taps * OC,
                nominal_macs_dilated=N * OC * taps * C * Op[0] * Op[1] * Op[2], V=V, O=O)
