"""Torch-facing helpers over the C ABI (argument marshalling only).

PyTorch provides device memory, streams and process groups; every step of the
C-K-S path runs in libcks.so's CUDA kernels.  Tensors are NHWC (activations)
and OHWI (filters), bfloat16 (CKS_BF16) or float32 (CKS_TF32); outputs fp32.
There is no CPU fallback: non-CUDA tensors raise.
"""
from __future__ import annotations

import contextlib

import torch

from . import _lib as L
from ._lib import CKS_BF16, CKS_TF32, make_geom

_WS: dict = {}


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return CKS_BF16
    if t.dtype == torch.float32:
        return CKS_TF32
    raise TypeError(f"unsupported dtype {t.dtype} (bfloat16 or float32)")


def _check_dev(*ts):
    for t in ts:
        if t is None:
            continue
        if not t.is_cuda:
            raise RuntimeError("C-K-S ops run on CUDA tensors only (no CPU fallback)")
        if not t.is_contiguous():
            raise RuntimeError("C-K-S ops take dense contiguous tensors")


def _stream_ptr(stream) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def _on(stream):
    """Allocate on the stream the kernels run on: the caching allocator then
    only hands a freed block to later work of that same stream (stream order),
    so a grown workspace or an output cannot be reused while queued kernels
    still read or write it."""
    return torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()


def _empty(shape, dtype, device, stream):
    with _on(stream):
        return torch.empty(shape, dtype=dtype, device=device)


def workspace(nbytes: int, device, stream=None) -> torch.Tensor | None:
    """Reusable per-(device, stream) scratch buffer (grown on demand; allocated
    on ``stream``, see _on)."""
    if nbytes == 0:
        return None
    key = (torch.device(device).index, _stream_ptr(stream))
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = _empty(max(nbytes, 1 << 20), torch.uint8, device, stream)
        _WS[key] = buf
    return buf


def _ws_args(ws):
    return (0, 0) if ws is None else (ws.data_ptr(), ws.numel())


def _pair(v):
    return (v, v) if isinstance(v, int) else tuple(v)


def geom_of(x_shape, w_shape, stride, padding):
    N, H, W, C = x_shape
    OC, FH, FW, C2 = w_shape
    if C != C2:
        raise ValueError(f"channel mismatch X {C} vs W {C2}")
    sh, sw = _pair(stride)
    ph, pw = _pair(padding)
    return make_geom(N, C, H, W, OC, FH, FW, sh, sw, ph, pw)


def conv2d_fwd(x, w, stride=1, padding=0, out=None, stream=None):
    """Y = conv2D(X, W) by ConvV2 (Eq (1), Alg. 1)."""
    _check_dev(x, w, out)
    dt = _dtype_code(x)
    g = geom_of(tuple(x.shape), tuple(w.shape), stride, padding)
    OH, OW = L.cks_output_shape(g)
    if out is None:
        out = _empty((g.N, OH, OW, g.OC), torch.float32, x.device, stream)
    ws = workspace(L.cks_workspace_size(g, dt, L.CKS_OP_FWD), x.device, stream)
    L.cks_conv2d_fwd(g, dt, x.data_ptr(), w.data_ptr(), out.data_ptr(), *_ws_args(ws), _stream_ptr(stream))
    return out


def ks_split(w, stride, x_hw=None, out=None, stream=None):
    """KS-deconv Stage1 (Alg. 2 Stage1): packed per-phase sub-filters."""
    _check_dev(w, out)
    dt = _dtype_code(w)
    OC, FH, FW, C = w.shape
    sh, sw = _pair(stride)
    H, W = x_hw if x_hw is not None else (FH, FW)
    g = make_geom(1, C, max(H, FH), max(W, FW), OC, FH, FW, sh, sw, 0, 0)
    nbytes = L.cks_ks_split_size(g, dt)
    if out is None:
        out = _empty(nbytes // w.element_size(), w.dtype, w.device, stream)
    L.cks_ks_split(g, dt, w.data_ptr(), out.data_ptr(), _stream_ptr(stream))
    return out


def deconv2d(dy, w, x_hw, stride=1, padding=0, c_packed=None, in_channels=None, out=None, stream=None,
             ks_mode="auto"):
    """dX = deconv2D(dY, W^rot180) by KS-deconv-V2 (Eq (2), Alg. 2/2B).
    ``x_hw`` = (I_H, I_W) of the forward input (output padding, reading c10).
    Pass ``c_packed`` (from ks_split) to skip Stage1; then ``w`` may be a
    shape-only tensor and is not read.  ``ks_mode`` (W given): "auto" (the
    library's choice), "stage1_free" (the GEMM reads W directly, no packed
    sub-filters), "stage1" (Stage1 into the workspace, then Stage2&3) or
    "multiphase" (narrow outputs: the phases stacked on the GEMM N dimension)."""
    _check_dev(dy, c_packed, out)
    dt = _dtype_code(dy)
    N, OH_, OW_, OC = dy.shape
    OC2, FH, FW, C = w.shape
    if OC != OC2:
        raise ValueError("dY channels != W out-channels")
    H, W = x_hw
    sh, sw = _pair(stride)
    ph, pw = _pair(padding)
    g = make_geom(N, C, H, W, OC, FH, FW, sh, sw, ph, pw)
    if L.cks_output_shape(g) != (OH_, OW_):
        raise ValueError("dY spatial shape does not match the geometry")
    if out is None:
        out = _empty((N, H, W, C), torch.float32, dy.device, stream)
    if c_packed is None:
        _check_dev(w)
        ws = workspace(L.cks_workspace_size(g, dt, L.CKS_OP_DECONV), dy.device, stream)
        wp, cp = w.data_ptr(), 0
    else:
        ws = workspace(L.cks_workspace_size(g, dt, L.CKS_OP_DECONV), dy.device, stream)
        wp, cp = 0, c_packed.data_ptr()
    mode = {"auto": L.CKS_KS_AUTO, "stage1_free": L.CKS_KS_STAGE1_FREE, "stage1": L.CKS_KS_STAGE1,
            "multiphase": L.CKS_KS_MULTIPHASE}[ks_mode]
    L.cks_deconv2d_ex(g, dt, dy.data_ptr(), wp or None, cp or None, out.data_ptr(), *_ws_args(ws),
                      _stream_ptr(stream), mode)
    return out


def dilated_wgrad(x, dy, filter_hw, stride=1, padding=0, gz=0, out=None, stream=None):
    """dW = dilated_conv2D(X, dY) by Sk-dilated-V2 (Eq (3), Alg. 3/3B)."""
    _check_dev(x, dy, out)
    dt = _dtype_code(x)
    N, H, W, C = x.shape
    OC = dy.shape[3]
    FH, FW = filter_hw
    sh, sw = _pair(stride)
    ph, pw = _pair(padding)
    g = make_geom(N, C, H, W, OC, FH, FW, sh, sw, ph, pw)
    if L.cks_output_shape(g) != tuple(dy.shape[1:3]):
        raise ValueError("dY spatial shape does not match the geometry")
    if out is None:
        out = _empty((OC, FH, FW, C), torch.float32, x.device, stream)
    ws = workspace(L.cks_workspace_size(g, dt, L.CKS_OP_WGRAD, gz), x.device, stream)
    L.cks_dilated_wgrad(g, dt, x.data_ptr(), dy.data_ptr(), out.data_ptr(), gz, *_ws_args(ws), _stream_ptr(stream))
    return out


# --------------------------------------------------------------- 3-D C-K-S
# NDHWC activations, OIDHW-as-[OC][FD][FH][FW][C] filters.
def _triple(v):
    return (v, v, v) if isinstance(v, int) else tuple(v)


def _geom3(x_shape, w_shape, stride, padding):
    N, D, H, W, C = x_shape
    OC, FD, FH, FW, C2 = w_shape
    if C != C2:
        raise ValueError("X channels != W in-channels")
    (sd, sh, sw), (pd, ph, pw) = _triple(stride), _triple(padding)
    return L.make_geom3(N, C, D, H, W, OC, FD, FH, FW, sd, sh, sw, pd, ph, pw)


def conv3d_fwd(x, w, stride=1, padding=0, out=None, stream=None):
    """Y = conv3D(X, W) by ConvV2 with trimmed windows on all three axes."""
    _check_dev(x, w, out)
    dt = _dtype_code(x)
    g = _geom3(tuple(x.shape), tuple(w.shape), stride, padding)
    OD, OH, OW = L.cks_output_shape3(g)
    if out is None:
        out = _empty((g.N, OD, OH, OW, g.OC), torch.float32, x.device, stream)
    ws = workspace(L.cks_workspace_size3(g, dt, L.CKS_OP_FWD), x.device, stream)
    L.cks_conv3d_fwd(g, dt, x.data_ptr(), w.data_ptr(), out.data_ptr(), *_ws_args(ws), _stream_ptr(stream))
    return out


def deconv3d(dy, w, x_dhw, stride=1, padding=0, out=None, stream=None):
    """dX = deconv3D(dY, W^rot180) by Stage1-free KS-deconv (sd*sh*sw phases)."""
    _check_dev(dy, w, out)
    dt = _dtype_code(dy)
    N = dy.shape[0]
    D, H, W = x_dhw
    g = _geom3((N, D, H, W, w.shape[4]), tuple(w.shape), stride, padding)
    if L.cks_output_shape3(g) != tuple(dy.shape[1:4]):
        raise ValueError("dY spatial shape does not match the geometry")
    if out is None:
        out = _empty((N, D, H, W, g.C), torch.float32, dy.device, stream)
    ws = workspace(L.cks_workspace_size3(g, dt, L.CKS_OP_DECONV), dy.device, stream)
    L.cks_deconv3d(g, dt, dy.data_ptr(), w.data_ptr(), out.data_ptr(), *_ws_args(ws), _stream_ptr(stream))
    return out


def dilated_wgrad3d(x, dy, filter_dhw, stride=1, padding=0, gz=0, out=None, stream=None):
    """dW = dilated_conv3D(X, dY) by Sk-dilated with leaping access on all axes."""
    _check_dev(x, dy, out)
    dt = _dtype_code(x)
    FD, FH, FW = filter_dhw
    g = _geom3(tuple(x.shape), (dy.shape[4], FD, FH, FW, x.shape[4]), stride, padding)
    if L.cks_output_shape3(g) != tuple(dy.shape[1:4]):
        raise ValueError("dY spatial shape does not match the geometry")
    if out is None:
        out = _empty((g.OC, FD, FH, FW, g.C), torch.float32, x.device, stream)
    ws = workspace(L.cks_workspace_size3(g, dt, L.CKS_OP_WGRAD, gz), x.device, stream)
    L.cks_dilated_wgrad3d(g, dt, x.data_ptr(), dy.data_ptr(), out.data_ptr(), gz, *_ws_args(ws),
                          _stream_ptr(stream))
    return out


# ----------------------------------------------------------------- KB-ZINS
# The zero-inserting / zero-padding formulation (include/cks.h KB-ZINS), on the
# same tensor-core kernels: a measurement baseline for the zeros C-K-S skips.
def zins_conv2d_fwd(x, w, stride=1, padding=0, out=None, stream=None):
    """Eq (1) on an explicitly zero-padded X (Fig. 1)."""
    _check_dev(x, w, out)
    dt = _dtype_code(x)
    g = geom_of(tuple(x.shape), tuple(w.shape), stride, padding)
    OH, OW = L.cks_output_shape(g)
    if out is None:
        out = _empty((g.N, OH, OW, g.OC), torch.float32, x.device, stream)
    ws = workspace(L.cks_zins_workspace_size(g, dt, L.CKS_OP_FWD), x.device, stream)
    L.cks_zins_conv2d_fwd(g, dt, x.data_ptr(), w.data_ptr(), out.data_ptr(), *_ws_args(ws), _stream_ptr(stream))
    return out


def zins_deconv2d(dy, w, x_hw, stride=1, padding=0, out=None, stream=None):
    """Eq (2) as P:114 states it: zero-inserted, padded dY conv W^rot180."""
    _check_dev(dy, w, out)
    dt = _dtype_code(dy)
    N, _, _, OC = dy.shape
    _, FH, FW, C = w.shape
    H, W = x_hw
    sh, sw = _pair(stride)
    ph, pw = _pair(padding)
    g = make_geom(N, C, H, W, OC, FH, FW, sh, sw, ph, pw)
    if L.cks_output_shape(g) != tuple(dy.shape[1:3]):
        raise ValueError("dY spatial shape does not match the geometry")
    if out is None:
        out = _empty((N, H, W, C), torch.float32, dy.device, stream)
    ws = workspace(L.cks_zins_workspace_size(g, dt, L.CKS_OP_DECONV), dy.device, stream)
    L.cks_zins_deconv2d(g, dt, dy.data_ptr(), w.data_ptr(), out.data_ptr(), *_ws_args(ws), _stream_ptr(stream))
    return out


def zins_wgrad(x, dy, filter_hw, stride=1, padding=0, out=None, stream=None):
    """Eq (3): the zero-inserted dY as the filter over padded X."""
    _check_dev(x, dy, out)
    dt = _dtype_code(x)
    N, H, W, C = x.shape
    OC = dy.shape[3]
    FH, FW = filter_hw
    sh, sw = _pair(stride)
    ph, pw = _pair(padding)
    g = make_geom(N, C, H, W, OC, FH, FW, sh, sw, ph, pw)
    if L.cks_output_shape(g) != tuple(dy.shape[1:3]):
        raise ValueError("dY spatial shape does not match the geometry")
    if out is None:
        out = _empty((OC, FH, FW, C), torch.float32, x.device, stream)
    ws = workspace(L.cks_zins_workspace_size(g, dt, L.CKS_OP_WGRAD), x.device, stream)
    L.cks_zins_wgrad(g, dt, x.data_ptr(), dy.data_ptr(), out.data_ptr(), *_ws_args(ws), _stream_ptr(stream))
    return out


# ------------------------------------------------------- autograd wrappers
# Conv-layer training through the three C-K-S operators: the
# forward of a convolution is ConvV2 (Eq 1) and its backward is KS-deconv
# (Eq 2, dX) + Sk-dilated (Eq 3, dW); a deconvolutional layer (the DCGAN
# generator) is the mirror image: forward KS-deconv, backward ConvV2 for
# the input gradient and Sk-dilated for the weight gradient.  The incoming
# gradient is rounded to the input dtype (bf16 / fp32) before the kernels.
class CKSConv2dFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, stride, padding):
        x, w = x.contiguous(), w.contiguous()  # backward's kernels take dense tensors too
        ctx.save_for_backward(x, w)
        ctx.stride, ctx.padding = _pair(stride), _pair(padding)
        return conv2d_fwd(x, w, ctx.stride, ctx.padding)

    @staticmethod
    def backward(ctx, gy):
        x, w = ctx.saved_tensors
        g = gy.to(x.dtype).contiguous()
        dx = dw = None
        if ctx.needs_input_grad[0]:
            dx = deconv2d(g, w, (x.shape[1], x.shape[2]), ctx.stride, ctx.padding).to(x.dtype)
        if ctx.needs_input_grad[1]:
            dw = dilated_wgrad(x, g, (w.shape[1], w.shape[2]), ctx.stride, ctx.padding).to(w.dtype)
        return dx, dw, None, None


class CKSConvTranspose2dFunction(torch.autograd.Function):
    """y = deconv2D(z, W^rot180) with W in the conv layout OHWI [O_C][F_H][F_W][I_C]
    (z has O_C channels, y has I_C channels and spatial extent ``out_hw``)."""

    @staticmethod
    def forward(ctx, z, w, out_hw, stride, padding):
        z, w = z.contiguous(), w.contiguous()  # backward's kernels take dense tensors too
        ctx.save_for_backward(z, w)
        ctx.stride, ctx.padding = _pair(stride), _pair(padding)
        return deconv2d(z, w, tuple(out_hw), ctx.stride, ctx.padding)

    @staticmethod
    def backward(ctx, gy):
        z, w = ctx.saved_tensors
        g = gy.to(z.dtype).contiguous()
        dz = dw = None
        if ctx.needs_input_grad[0]:
            dz = conv2d_fwd(g, w, ctx.stride, ctx.padding).to(z.dtype)
        if ctx.needs_input_grad[1]:
            dw = dilated_wgrad(g, z, (w.shape[1], w.shape[2]), ctx.stride, ctx.padding).to(w.dtype)
        return dz, dw, None, None, None


def cks_conv2d(x, w, stride=1, padding=0):
    return CKSConv2dFunction.apply(x, w, stride, padding)


def cks_conv_transpose2d(z, w, out_hw, stride=1, padding=0):
    return CKSConvTranspose2dFunction.apply(z, w, out_hw, stride, padding)
