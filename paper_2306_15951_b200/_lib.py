"""ctypes binding of libcks.so (include/cks.h) -- argument marshalling only.

Every function here has the name of the C entry point it calls and takes
plain integers / pointers.  All compute runs in the CUDA kernels behind the C
ABI; there is no CPU fallback: if the library is missing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# CKS_EXPERIMENTS=1 loads the experiments build (libcks_exp.so: environment
# knobs for tools/ sweeps); the product path loads libcks.so, which has none
LIB_PATH = os.path.join(_PKG, "libcks_exp.so" if os.environ.get("CKS_EXPERIMENTS") == "1" else "libcks.so")

CKS_TF32, CKS_BF16 = 0, 1
CKS_OP_FWD, CKS_OP_DECONV, CKS_OP_WGRAD = 0, 1, 2
STATUS = {0: "CKS_OK", 1: "CKS_ERR_NULL", 2: "CKS_ERR_GEOMETRY", 3: "CKS_ERR_UNSUPPORTED",
          4: "CKS_ERR_ALIGNMENT", 5: "CKS_ERR_WORKSPACE", 6: "CKS_ERR_CUDA", 7: "CKS_ERR_CAPACITY"}

# Every symbol include/cks.h declares (tests check the .so exports all of them).
EXPORTS = ("cks_output_shape", "cks_workspace_size", "cks_choose_gz", "cks_conv2d_fwd", "cks_ks_split_size",
           "cks_ks_split", "cks_deconv2d", "cks_dilated_wgrad", "cks_axis_table", "cks_op_counts",
           "cks_launch_count", "cks_status_string", "cks_version", "cks_zins_workspace_size",
           "cks_zins_conv2d_fwd", "cks_zins_deconv2d", "cks_zins_wgrad", "cks_plan_describe", "cks_deconv2d_ex",
           "cks_padding_macs", "cks_output_shape3", "cks_workspace_size3", "cks_op_counts3", "cks_conv3d_fwd",
           "cks_deconv3d", "cks_dilated_wgrad3d", "cks_ar_recv_bytes", "cks_dilated_wgrad_allreduce", "cks_ipc_export",
           "cks_ipc_import", "cks_ipc_close", "cks_dilated_wgrad_allreduce_emulated")


class CksError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {STATUS.get(status, status)} ({_string(status)})")


class cks_geom(C.Structure):
    _fields_ = [("N", C.c_int64), ("C", C.c_int64), ("H", C.c_int64), ("W", C.c_int64), ("OC", C.c_int64),
                ("FH", C.c_int64), ("FW", C.c_int64), ("sh", C.c_int32), ("sw", C.c_int32), ("ph", C.c_int32),
                ("pw", C.c_int32), ("dh", C.c_int32), ("dw", C.c_int32)]


CKS_AR_MAX_RANKS = 8
CKS_OP_WGRAD_AR = 3


class cks_ar_group(C.Structure):
    """include/cks.h cks_ar_group: the peers' buffers of one fused wgrad + all-reduce."""
    _fields_ = [("world", C.c_int32), ("rank", C.c_int32), ("ctas", C.c_int32),
                ("recv", C.c_void_p * CKS_AR_MAX_RANKS), ("out", C.c_void_p * CKS_AR_MAX_RANKS),
                ("flag", C.c_void_p * CKS_AR_MAX_RANKS), ("count", C.c_void_p), ("err", C.c_void_p)]


class cks_geom3(C.Structure):
    """include/cks.h cks_geom3 (3-D C-K-S)."""
    _fields_ = [(n, C.c_int64) for n in ("N", "C", "D", "H", "W", "OC", "FD", "FH", "FW")] + \
               [(n, C.c_int32) for n in ("sd", "sh", "sw", "pd", "ph", "pw")]


def make_geom3(N, C_, D, H, W, OC, FD, FH, FW, sd, sh, sw, pd, ph, pw) -> cks_geom3:
    return cks_geom3(N, C_, D, H, W, OC, FD, FH, FW, sd, sh, sw, pd, ph, pw)


class cks_ipc_handle(C.Structure):
    _fields_ = [("bytes", C.c_ubyte * 72)]


def make_geom(N, C_, H, W, OC, FH, FW, sh, sw, ph, pw, dh=1, dw=1) -> cks_geom:
    return cks_geom(N, C_, H, W, OC, FH, FW, sh, sw, ph, pw, dh, dw)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libcks.so not built ({LIB_PATH}); run python -m paper_2306_15951_b200.build "
                               "or __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        G = C.POINTER(cks_geom)
        G3 = C.POINTER(cks_geom3)
        vp, sz = C.c_void_p, C.c_size_t
        sig = {
            "cks_output_shape": (C.c_int, [G, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
            "cks_workspace_size": (C.c_int, [G, C.c_int, C.c_int, C.c_int, C.POINTER(sz)]),
            "cks_choose_gz": (C.c_int, [G, C.c_int, C.POINTER(C.c_int)]),
            "cks_conv2d_fwd": (C.c_int, [G, C.c_int, vp, vp, vp, vp, sz, vp]),
            "cks_ks_split_size": (C.c_int, [G, C.c_int, C.POINTER(sz)]),
            "cks_ks_split": (C.c_int, [G, C.c_int, vp, vp, vp]),
            "cks_deconv2d": (C.c_int, [G, C.c_int, vp, vp, vp, vp, vp, sz, vp]),
            "cks_deconv2d_ex": (C.c_int, [G, C.c_int, vp, vp, vp, vp, vp, sz, vp, C.c_int]),
            "cks_dilated_wgrad": (C.c_int, [G, C.c_int, vp, vp, vp, C.c_int, vp, sz, vp]),
            "cks_axis_table": (C.c_int, [C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_int,
                                         C.POINTER(C.c_int64), sz, C.POINTER(sz)]),
            "cks_op_counts": (C.c_int, [G, C.c_int, C.POINTER(C.c_int64)]),
            "cks_launch_count": (C.c_int, [G, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]),
            "cks_zins_workspace_size": (C.c_int, [G, C.c_int, C.c_int, C.POINTER(sz)]),
            "cks_zins_conv2d_fwd": (C.c_int, [G, C.c_int, vp, vp, vp, vp, sz, vp]),
            "cks_zins_deconv2d": (C.c_int, [G, C.c_int, vp, vp, vp, vp, sz, vp]),
            "cks_zins_wgrad": (C.c_int, [G, C.c_int, vp, vp, vp, vp, sz, vp]),
            "cks_plan_describe": (C.c_int, [G, C.c_int, C.c_int, C.c_int, C.c_char_p, sz, C.POINTER(sz)]),
            "cks_padding_macs": (C.c_int, [G, C.c_int, C.c_int, C.POINTER(C.c_int64)]),
            "cks_output_shape3": (C.c_int, [G3, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
            "cks_workspace_size3": (C.c_int, [G3, C.c_int, C.c_int, C.c_int, C.POINTER(sz)]),
            "cks_op_counts3": (C.c_int, [G3, C.POINTER(C.c_int64)]),
            "cks_conv3d_fwd": (C.c_int, [G3, C.c_int, vp, vp, vp, vp, sz, vp]),
            "cks_deconv3d": (C.c_int, [G3, C.c_int, vp, vp, vp, vp, sz, vp]),
            "cks_dilated_wgrad3d": (C.c_int, [G3, C.c_int, vp, vp, vp, C.c_int, vp, sz, vp]),
            "cks_ar_recv_bytes": (C.c_int, [G, C.c_int32, C.POINTER(sz)]),
            "cks_dilated_wgrad_allreduce": (C.c_int, [G, C.c_int, vp, vp, vp, C.c_int, vp, sz,
                                                      C.POINTER(cks_ar_group), vp]),
            "cks_dilated_wgrad_allreduce_emulated": (C.c_int, [C.c_int32, G, C.c_int, C.POINTER(vp), C.POINTER(vp),
                                                               C.POINTER(vp), C.c_int, C.POINTER(vp), C.POINTER(sz),
                                                               C.POINTER(cks_ar_group), vp]),
            "cks_ipc_export": (C.c_int, [vp, C.POINTER(cks_ipc_handle)]),
            "cks_ipc_import": (C.c_int, [C.POINTER(cks_ipc_handle), C.POINTER(vp)]),
            "cks_ipc_close": (C.c_int, [vp]),
            "cks_status_string": (C.c_char_p, [C.c_int]),
            "cks_version": (C.c_int, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def _string(status: int) -> str:
    try:
        return lib().cks_status_string(status).decode()
    except Exception:  # pragma: no cover
        return "?"


def _check(st: int, where: str):
    if st != 0:
        raise CksError(st, where)


# ------------------------------------------------------------ thin wrappers
def cks_version() -> int:
    return lib().cks_version()


def cks_output_shape(g: cks_geom):
    oh, ow = C.c_int64(), C.c_int64()
    _check(lib().cks_output_shape(C.byref(g), C.byref(oh), C.byref(ow)), "cks_output_shape")
    return oh.value, ow.value


def cks_workspace_size(g: cks_geom, dtype: int, op: int, gz: int = 0) -> int:
    b = C.c_size_t()
    _check(lib().cks_workspace_size(C.byref(g), dtype, op, gz, C.byref(b)), "cks_workspace_size")
    return b.value


def cks_choose_gz(g: cks_geom, dtype: int) -> int:
    v = C.c_int()
    _check(lib().cks_choose_gz(C.byref(g), dtype, C.byref(v)), "cks_choose_gz")
    return v.value


def cks_ks_split_size(g: cks_geom, dtype: int) -> int:
    b = C.c_size_t()
    _check(lib().cks_ks_split_size(C.byref(g), dtype, C.byref(b)), "cks_ks_split_size")
    return b.value


def cks_conv2d_fwd(g, dtype, x_ptr, w_ptr, y_ptr, ws_ptr, ws_bytes, stream):
    _check(lib().cks_conv2d_fwd(C.byref(g), dtype, x_ptr, w_ptr, y_ptr, ws_ptr, ws_bytes, stream), "cks_conv2d_fwd")


def cks_ks_split(g, dtype, w_ptr, c_ptr, stream):
    _check(lib().cks_ks_split(C.byref(g), dtype, w_ptr, c_ptr, stream), "cks_ks_split")


def cks_deconv2d(g, dtype, dy_ptr, w_ptr, c_ptr, dx_ptr, ws_ptr, ws_bytes, stream):
    _check(lib().cks_deconv2d(C.byref(g), dtype, dy_ptr, w_ptr, c_ptr, dx_ptr, ws_ptr, ws_bytes, stream),
           "cks_deconv2d")


CKS_KS_AUTO, CKS_KS_STAGE1_FREE, CKS_KS_STAGE1, CKS_KS_MULTIPHASE = 0, 1, 2, 3


def cks_deconv2d_ex(g, dtype, dy_ptr, w_ptr, c_ptr, dx_ptr, ws_ptr, ws_bytes, stream, mode):
    _check(lib().cks_deconv2d_ex(C.byref(g), dtype, dy_ptr, w_ptr, c_ptr, dx_ptr, ws_ptr, ws_bytes, stream, mode),
           "cks_deconv2d_ex")


# ------------------------------------------------------------------ 3-D C-K-S
def cks_output_shape3(g: cks_geom3):
    od, oh, ow = C.c_int64(), C.c_int64(), C.c_int64()
    _check(lib().cks_output_shape3(C.byref(g), C.byref(od), C.byref(oh), C.byref(ow)), "cks_output_shape3")
    return od.value, oh.value, ow.value


def cks_workspace_size3(g: cks_geom3, dtype: int, op: int, gz: int = 0) -> int:
    b = C.c_size_t()
    _check(lib().cks_workspace_size3(C.byref(g), dtype, op, gz, C.byref(b)), "cks_workspace_size3")
    return b.value


def cks_op_counts3(g: cks_geom3) -> dict:
    out = (C.c_int64 * 4)()
    _check(lib().cks_op_counts3(C.byref(g), out), "cks_op_counts3")
    return {"zero_free_macs": out[0], "VD": out[1], "VH": out[2], "VW": out[3]}


def cks_conv3d_fwd(g, dtype, x_ptr, w_ptr, y_ptr, ws_ptr, ws_bytes, stream):
    _check(lib().cks_conv3d_fwd(C.byref(g), dtype, x_ptr, w_ptr, y_ptr, ws_ptr, ws_bytes, stream), "cks_conv3d_fwd")


def cks_deconv3d(g, dtype, dy_ptr, w_ptr, dx_ptr, ws_ptr, ws_bytes, stream):
    _check(lib().cks_deconv3d(C.byref(g), dtype, dy_ptr, w_ptr, dx_ptr, ws_ptr, ws_bytes, stream), "cks_deconv3d")


def cks_dilated_wgrad3d(g, dtype, x_ptr, dy_ptr, dw_ptr, gz, ws_ptr, ws_bytes, stream):
    _check(lib().cks_dilated_wgrad3d(C.byref(g), dtype, x_ptr, dy_ptr, dw_ptr, gz, ws_ptr, ws_bytes, stream),
           "cks_dilated_wgrad3d")


def cks_ar_recv_bytes(g: cks_geom, world: int) -> int:
    v = C.c_size_t()
    _check(lib().cks_ar_recv_bytes(C.byref(g), world, C.byref(v)), "cks_ar_recv_bytes")
    return v.value


def cks_dilated_wgrad_allreduce(g, dtype, x_ptr, dy_ptr, dw_ptr, gz, ws_ptr, ws_bytes, grp: cks_ar_group, stream):
    _check(lib().cks_dilated_wgrad_allreduce(C.byref(g), dtype, x_ptr, dy_ptr, dw_ptr, gz, ws_ptr, ws_bytes,
                                             C.byref(grp), stream), "cks_dilated_wgrad_allreduce")


def cks_dilated_wgrad_allreduce_emulated(geoms, dtype, x_ptrs, dy_ptrs, dw_ptrs, gz, ws_ptrs, ws_bytes, grps,
                                         stream):
    """All `len(geoms)` ranks on this GPU: per-rank lists; one cooperative reduce launch."""
    w = len(geoms)
    GA, PA, SA, RA = cks_geom * w, C.c_void_p * w, C.c_size_t * w, cks_ar_group * w
    _check(lib().cks_dilated_wgrad_allreduce_emulated(w, GA(*geoms), dtype, PA(*x_ptrs), PA(*dy_ptrs), PA(*dw_ptrs),
                                                      gz, PA(*ws_ptrs), SA(*ws_bytes), RA(*grps), stream),
           "cks_dilated_wgrad_allreduce_emulated")


def cks_ipc_export(ptr: int) -> bytes:
    h = cks_ipc_handle()
    _check(lib().cks_ipc_export(ptr, C.byref(h)), "cks_ipc_export")
    return bytes(h.bytes)


def cks_ipc_import(handle: bytes) -> int:
    h = cks_ipc_handle()
    C.memmove(h.bytes, handle, 72)
    p = C.c_void_p()
    _check(lib().cks_ipc_import(C.byref(h), C.byref(p)), "cks_ipc_import")
    return p.value


def cks_ipc_close(ptr: int):
    _check(lib().cks_ipc_close(ptr), "cks_ipc_close")


def cks_dilated_wgrad(g, dtype, x_ptr, dy_ptr, dw_ptr, gz, ws_ptr, ws_bytes, stream):
    _check(lib().cks_dilated_wgrad(C.byref(g), dtype, x_ptr, dy_ptr, dw_ptr, gz, ws_ptr, ws_bytes, stream),
           "cks_dilated_wgrad")


def cks_axis_table(I: int, F: int, s: int, p: int, table: int) -> list:
    n = C.c_size_t()
    st = lib().cks_axis_table(I, F, s, p, table, None, 0, C.byref(n))
    if st not in (0, 7):
        _check(st, "cks_axis_table")
    buf = (C.c_int64 * max(n.value, 1))()
    _check(lib().cks_axis_table(I, F, s, p, table, buf, n.value, C.byref(n)), "cks_axis_table")
    return list(buf[:n.value])


def cks_op_counts(g: cks_geom, dtype: int = CKS_BF16) -> dict:
    out = (C.c_int64 * 8)()
    _check(lib().cks_op_counts(C.byref(g), dtype, out), "cks_op_counts")
    keys = ("zero_free_macs", "VH", "VW", "T_conv", "T_deconv", "T_dilated", "issued_macs_fwd", "tiles_fwd")
    return dict(zip(keys, list(out)))


def cks_launch_count(g: cks_geom, dtype: int, op: int, gz: int = 0, c_packed_given: bool = False) -> int:
    v = C.c_int()
    _check(lib().cks_launch_count(C.byref(g), dtype, op, gz, int(c_packed_given), C.byref(v)), "cks_launch_count")
    return v.value


def cks_plan_describe(g: cks_geom, dtype: int, op: int, gz: int = 0) -> str:
    n = C.c_size_t()
    st = lib().cks_plan_describe(C.byref(g), dtype, op, gz, None, 0, C.byref(n))
    if st not in (0, 7):
        _check(st, "cks_plan_describe")
    buf = C.create_string_buffer(n.value)
    _check(lib().cks_plan_describe(C.byref(g), dtype, op, gz, buf, n.value, C.byref(n)), "cks_plan_describe")
    return buf.value.decode()


def plan_dict(g: cks_geom, dtype: int, op: int, gz: int = 0) -> dict:
    """cks_plan_describe parsed: {'kind': ..., key: value (str)}."""
    parts = cks_plan_describe(g, dtype, op, gz).split()
    d = {"kind": parts[0]}
    d.update(kv.split("=", 1) for kv in parts[1:])
    return d


def cks_padding_macs(g: cks_geom, dtype: int, op: int) -> int:
    v = C.c_int64()
    _check(lib().cks_padding_macs(C.byref(g), dtype, op, C.byref(v)), "cks_padding_macs")
    return v.value


# ------------------------------------------------ KB-ZINS (measurement baseline)
def cks_zins_workspace_size(g: cks_geom, dtype: int, op: int) -> int:
    b = C.c_size_t()
    _check(lib().cks_zins_workspace_size(C.byref(g), dtype, op, C.byref(b)), "cks_zins_workspace_size")
    return b.value


def cks_zins_conv2d_fwd(g, dtype, x_ptr, w_ptr, y_ptr, ws_ptr, ws_bytes, stream):
    _check(lib().cks_zins_conv2d_fwd(C.byref(g), dtype, x_ptr, w_ptr, y_ptr, ws_ptr, ws_bytes, stream),
           "cks_zins_conv2d_fwd")


def cks_zins_deconv2d(g, dtype, dy_ptr, w_ptr, dx_ptr, ws_ptr, ws_bytes, stream):
    _check(lib().cks_zins_deconv2d(C.byref(g), dtype, dy_ptr, w_ptr, dx_ptr, ws_ptr, ws_bytes, stream),
           "cks_zins_deconv2d")


def cks_zins_wgrad(g, dtype, x_ptr, dy_ptr, dw_ptr, ws_ptr, ws_bytes, stream):
    _check(lib().cks_zins_wgrad(C.byref(g), dtype, x_ptr, dy_ptr, dw_ptr, ws_ptr, ws_bytes, stream),
           "cks_zins_wgrad")
