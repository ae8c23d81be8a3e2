"""Python binding of libfgf.so, the B200-native Fast Guided Filter (arXiv 1505.00996).

Argument marshalling only: every step of Alg. 2 runs in the CUDA
kernels of csrc/ behind the C ABI of include/fgf.h.  The binding has the C names
(fgf_filter, fgf_filter_ws, fgf_filter_host, fgf_coefficients, fgf_upsample_output,
fgf_workspace_bytes, fgf_status_str, fgf_last_launch_count) and accepts torch tensors
(or raw integer addresses) for the buffers.  There is no CPU fallback: importing this
package without the built library raises ImportError.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, os.environ.get("FGF_LIB_NAME", "libfgf.so"))   # (A/B builds)

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
                      "there is no fallback implementation")

_lib = ctypes.CDLL(LIB_PATH)

FGF_OK = 0
FGF_ERR_PARAM = 1
FGF_ERR_SHAPE = 2
FGF_ERR_NULL = 3
FGF_ERR_ALIAS = 4
FGF_ERR_ALIGN = 5
FGF_ERR_CUDA = 6
FGF_ERR_NOMEM = 7
FGF_ERR_NCCL = 8
FGF_ERR_UNSUPPORTED = 9
FGF_ERR_DEVICE = 10
FGF_F32 = 0
FGF_F16 = 1
FGF_BF16 = 2
FGF_U8 = 3
FGF_BAND_SINGLE = 0
FGF_BAND_TWO_STEP = 1
FGF_GUIDE_SELF = 0
FGF_GUIDE_LUMA = 1
FGF_SUB_NEAREST = 0
FGF_SUB_BILINEAR = 1

# Every symbol include/fgf.h declares (tests check the library exports each one).
EXPORTS = ("fgf_filter", "fgf_workspace_bytes", "fgf_filter_ws", "fgf_filter_host",
           "fgf_coefficients", "fgf_upsample_output", "fgf_last_launch_count", "fgf_status_str",
           "fgf_version", "fgf_profile_enable", "fgf_profile_read", "fgf_subsample",
           "fgf_lowres_workspace_bytes", "fgf_lowres_mean", "fgf_upsample_output_rows",
           "fgf_enhance_ws", "fgf_band_workspace_bytes", "fgf_filter_band", "fgf_nccl_unique_id",
           "fgf_nccl_comm_init", "fgf_nccl_comm_destroy", "fgf_bands_loopback_workspace_bytes",
           "fgf_filter_bands_loopback", "fgf_workspace_bytes_ex", "fgf_filter_ex_ws",
           "fgf_filter_band_ex", "fgf_joint_workspace_bytes", "fgf_filter_joint_ws",
           "fgf_nccl_check", "fgf_band_geometry", "fgf_enhance_workspace_bytes",
           "fgf_enhance_ex_ws", "fgf_filter_host_input_bytes",
           "fgf_filter_host_ex")
KERNEL_KINDS = ("subsample", "stats_coef", "box_ab", "upsample_output", "lowres_fused",
                "wide_fused", "tiny_fused")

_P = ctypes.c_void_p
_i, _d, _sz = ctypes.c_int, ctypes.c_double, ctypes.c_size_t
_GEOM = [_i, _i, _i, _i, _i, _i, _d, _i, _i]  # batch H W C_I C_p r eps s sub_mode
_lib.fgf_filter.argtypes = [_P, _P, _P] + _GEOM
_lib.fgf_filter.restype = _i
_lib.fgf_filter_ws.argtypes = [_P, _P, _P] + _GEOM + [_P, _sz, _P]
_lib.fgf_filter_ws.restype = _i
_lib.fgf_filter_host.argtypes = [_P, _P, _P] + _GEOM + [_i]
_lib.fgf_filter_host.restype = _i
_lib.fgf_filter_host_input_bytes.argtypes = [_i] * 10
_lib.fgf_filter_host_ex.argtypes = [_P, _P, _P] + _GEOM + [_i, _i]
_lib.fgf_filter_host_ex.restype = _i
_lib.fgf_filter_host_input_bytes.restype = _sz
_lib.fgf_coefficients.argtypes = [_P, _P, _P] + _GEOM + [_P, _sz, _P]
_lib.fgf_coefficients.restype = _i
_lib.fgf_upsample_output.argtypes = [_P, _P, _P, _i, _i, _i, _i, _i, _i, _P]
_lib.fgf_upsample_output.restype = _i
_lib.fgf_workspace_bytes.argtypes = [_i, _i, _i, _i, _i, _i, _i]
_lib.fgf_workspace_bytes.restype = _sz
_lib.fgf_last_launch_count.argtypes = []
_lib.fgf_last_launch_count.restype = _i
_lib.fgf_status_str.argtypes = [_i]
_lib.fgf_status_str.restype = ctypes.c_char_p
_lib.fgf_profile_enable.argtypes = [_i]
_lib.fgf_profile_enable.restype = _i
_lib.fgf_profile_read.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int), _i]
_lib.fgf_profile_read.restype = _i
_lib.fgf_subsample.argtypes = [_P, _P, _i, _i, _i, _i, _i, _P]
_lib.fgf_subsample.restype = _i
_lib.fgf_lowres_workspace_bytes.argtypes = [_i, _i, _i, _i, _i]
_lib.fgf_lowres_workspace_bytes.restype = _sz
_lib.fgf_lowres_mean.argtypes = [_P, _P, _P, _i, _i, _i, _i, _i, _i, _d, _P, _sz, _P]
_lib.fgf_lowres_mean.restype = _i
_lib.fgf_upsample_output_rows.argtypes = [_P, _P, _P] + [_i] * 11 + [_P]
_lib.fgf_upsample_output_rows.restype = _i
_lib.fgf_enhance_ws.argtypes = [_P, _P, _i, _i, _i, _i, _i, _d, _i, _i, _d, _P, _sz, _P]
_lib.fgf_enhance_ws.restype = _i
_lib.fgf_band_workspace_bytes.argtypes = [_i] * 9
_lib.fgf_band_workspace_bytes.restype = _sz
_lib.fgf_filter_band.argtypes = [_P, _P, _P] + [_i] * 7 + [_d, _i, _i, _P, _i, _i, _P, _sz, _P]
_lib.fgf_filter_band.restype = _i
_lib.fgf_nccl_unique_id.argtypes = [_P]
_lib.fgf_nccl_unique_id.restype = _i
_lib.fgf_nccl_comm_init.argtypes = [ctypes.POINTER(ctypes.c_void_p), _P, _i, _i]
_lib.fgf_nccl_comm_init.restype = _i
_lib.fgf_nccl_check.argtypes = [_P]
_lib.fgf_nccl_check.restype = _i
_lib.fgf_nccl_comm_destroy.argtypes = [_P]
_lib.fgf_nccl_comm_destroy.restype = _i
_lib.fgf_bands_loopback_workspace_bytes.argtypes = [_i] * 7
_lib.fgf_bands_loopback_workspace_bytes.restype = _sz
_lib.fgf_filter_bands_loopback.argtypes = [_P, _P, _P] + [_i] * 5 + [_d, _i, _i, _i, _i, _P, _sz, _P]
_lib.fgf_filter_band_ex.argtypes = [_P, _P, _P] + [_i] * 7 + [_d, _i, _i, _i, _P, _i, _i, _P, _sz, _P]
_lib.fgf_filter_band_ex.restype = _i
_lib.fgf_filter_bands_loopback.restype = _i
_lib.fgf_workspace_bytes_ex.argtypes = [_i] * 8
_lib.fgf_workspace_bytes_ex.restype = _sz
_lib.fgf_filter_ex_ws.argtypes = [_P, _P, _P] + _GEOM + [_i, _P, _sz, _P]
_lib.fgf_filter_ex_ws.restype = _i
_lib.fgf_joint_workspace_bytes.argtypes = [_i] * 7
_lib.fgf_joint_workspace_bytes.restype = _sz
_lib.fgf_filter_joint_ws.argtypes = [_P, _P, _P] + _GEOM + [_P, _sz, _P]
_lib.fgf_filter_joint_ws.restype = _i
_lib.fgf_band_geometry.argtypes = [_i, _i, _i, _i, _i, _i, ctypes.POINTER(ctypes.c_int)]
_lib.fgf_band_geometry.restype = _i
_lib.fgf_enhance_workspace_bytes.argtypes = [_i] * 7
_lib.fgf_enhance_workspace_bytes.restype = _sz
_lib.fgf_enhance_ex_ws.argtypes = [_P, _P] + [_i] * 5 + [_d, _i, _i, _d, _i, _P, _sz, _P]
_lib.fgf_enhance_ex_ws.restype = _i
_lib.fgf_version.argtypes = []
_lib.fgf_version.restype = ctypes.c_char_p


class FGFError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: {fgf_status_str(status)} (status {status})")
        self.status = status


def _addr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):  # numpy
        return x.ctypes.data
    raise TypeError(f"cannot take the address of {type(x)}")


def _stream(st):
    if st is None:
        return None
    if isinstance(st, int):
        return st
    return st.cuda_stream


def _check(rc: int, where: str) -> None:
    if rc != FGF_OK:
        raise FGFError(rc, where)


def fgf_status_str(status: int) -> str:
    return _lib.fgf_status_str(status).decode()


def fgf_version() -> str:
    return _lib.fgf_version().decode()


def fgf_last_launch_count() -> int:
    return _lib.fgf_last_launch_count()


def fgf_profile_enable(on: bool) -> None:
    _lib.fgf_profile_enable(1 if on else 0)


def fgf_profile_read():
    """{kind: (total_ms, launches)} for the launches recorded since fgf_profile_enable."""
    nk = len(KERNEL_KINDS)
    ms = (ctypes.c_double * nk)()
    n = (ctypes.c_int * nk)()
    k = _lib.fgf_profile_read(ms, n, nk)
    if k < 0:
        raise FGFError(-k, "fgf_profile_read")
    return {KERNEL_KINDS[i]: (ms[i], n[i]) for i in range(k)}


def fgf_workspace_bytes(batch, H, W, C_I, C_p, r, s) -> int:
    return _lib.fgf_workspace_bytes(batch, H, W, C_I, C_p, r, s)


def fgf_filter(I, p, q, batch, H, W, C_I, C_p, r, eps, s, sub_mode=FGF_SUB_NEAREST, check=True):
    rc = _lib.fgf_filter(_addr(I), _addr(p), _addr(q), batch, H, W, C_I, C_p, r, float(eps), s,
                         sub_mode)
    if check:
        _check(rc, "fgf_filter")
    return rc


def fgf_filter_ws(I, p, q, batch, H, W, C_I, C_p, r, eps, s, sub_mode, workspace, ws_bytes,
                  stream=None, check=True):
    rc = _lib.fgf_filter_ws(_addr(I), _addr(p), _addr(q), batch, H, W, C_I, C_p, r, float(eps),
                            s, sub_mode, _addr(workspace), ws_bytes, _stream(stream))
    if check:
        _check(rc, "fgf_filter_ws")
    return rc


def fgf_filter_host(I, p, q, batch, H, W, C_I, C_p, r, eps, s, sub_mode=FGF_SUB_NEAREST,
                    device=0, check=True):
    rc = _lib.fgf_filter_host(_addr(I), _addr(p), _addr(q), batch, H, W, C_I, C_p, r, float(eps),
                              s, sub_mode, device)
    if check:
        _check(rc, "fgf_filter_host")
    return rc


def fgf_filter_host_input_bytes(batch, H, W, C_I, C_p, r, s, sub_mode=FGF_SUB_NEAREST,
                                dtype=FGF_F32, self_guided=False):
    return int(_lib.fgf_filter_host_input_bytes(batch, H, W, C_I, C_p, r, s, sub_mode, dtype,
                                                1 if self_guided else 0))


def fgf_filter_host_ex(I, p, q, batch, H, W, C_I, C_p, r, eps, s, sub_mode, dtype, device=0,
                       check=True):
    rc = _lib.fgf_filter_host_ex(_addr(I), _addr(p), _addr(q), batch, H, W, C_I, C_p, r,
                                 float(eps), s, sub_mode, dtype, device)
    if check:
        _check(rc, "fgf_filter_host_ex")
    return rc


def fgf_coefficients(I, p, mean_ab, batch, H, W, C_I, C_p, r, eps, s, sub_mode, workspace,
                     ws_bytes, stream=None, check=True):
    rc = _lib.fgf_coefficients(_addr(I), _addr(p), _addr(mean_ab), batch, H, W, C_I, C_p, r,
                               float(eps), s, sub_mode, _addr(workspace), ws_bytes,
                               _stream(stream))
    if check:
        _check(rc, "fgf_coefficients")
    return rc


def fgf_upsample_output(I, mean_ab, q, batch, H, W, C_I, C_p, s, stream=None, check=True):
    rc = _lib.fgf_upsample_output(_addr(I), _addr(mean_ab), _addr(q), batch, H, W, C_I, C_p, s,
                                  _stream(stream))
    if check:
        _check(rc, "fgf_upsample_output")
    return rc


def fgf_subsample(src, dst, planes, H, W, s, sub_mode=FGF_SUB_NEAREST, stream=None, check=True):
    rc = _lib.fgf_subsample(_addr(src), _addr(dst), planes, H, W, s, sub_mode, _stream(stream))
    if check:
        _check(rc, "fgf_subsample")
    return rc


def fgf_lowres_workspace_bytes(batch, h, w, C_I, C_p) -> int:
    return _lib.fgf_lowres_workspace_bytes(batch, h, w, C_I, C_p)


def fgf_lowres_mean(Is, ps, mean_ab, batch, h, w, C_I, C_p, r_low, eps, workspace, ws_bytes,
                    stream=None, check=True):
    rc = _lib.fgf_lowres_mean(_addr(Is), _addr(ps), _addr(mean_ab), batch, h, w, C_I, C_p, r_low,
                              float(eps), _addr(workspace), ws_bytes, _stream(stream))
    if check:
        _check(rc, "fgf_lowres_mean")
    return rc


def fgf_upsample_output_rows(I, mean_ab, q, batch, rows, W, C_I, C_p, H_total, h_total, w, Y0,
                             y0_maps, h_maps, stream=None, check=True):
    rc = _lib.fgf_upsample_output_rows(_addr(I), _addr(mean_ab), _addr(q), batch, rows, W, C_I, C_p,
                                       H_total, h_total, w, Y0, y0_maps, h_maps, _stream(stream))
    if check:
        _check(rc, "fgf_upsample_output_rows")
    return rc


def fgf_enhance_ws(I, out, batch, H, W, C, r, eps, s, sub_mode, gain, workspace, ws_bytes,
                   stream=None, check=True):
    rc = _lib.fgf_enhance_ws(_addr(I), _addr(out), batch, H, W, C, r, float(eps), s, sub_mode,
                             float(gain), _addr(workspace), ws_bytes, _stream(stream))
    if check:
        _check(rc, "fgf_enhance_ws")
    return rc


def fgf_workspace_bytes_ex(batch, H, W, C_I, C_p, r, s, dtype) -> int:
    return _lib.fgf_workspace_bytes_ex(batch, H, W, C_I, C_p, r, s, dtype)


def fgf_filter_ex_ws(I, p, q, batch, H, W, C_I, C_p, r, eps, s, sub_mode, dtype, workspace,
                     ws_bytes, stream=None, check=True):
    rc = _lib.fgf_filter_ex_ws(_addr(I), _addr(p), _addr(q), batch, H, W, C_I, C_p, r,
                               float(eps), s, sub_mode, dtype, _addr(workspace), ws_bytes,
                               _stream(stream))
    if check:
        _check(rc, "fgf_filter_ex_ws")
    return rc


def fgf_joint_workspace_bytes(batch, H, W, C_I, C_p, r, s) -> int:
    return _lib.fgf_joint_workspace_bytes(batch, H, W, C_I, C_p, r, s)


def fgf_filter_joint_ws(I, p_low, q, batch, H, W, C_I, C_p, r, eps, s, sub_mode, workspace,
                        ws_bytes, stream=None, check=True):
    rc = _lib.fgf_filter_joint_ws(_addr(I), _addr(p_low), _addr(q), batch, H, W, C_I, C_p, r,
                                  float(eps), s, sub_mode, _addr(workspace), ws_bytes,
                                  _stream(stream))
    if check:
        _check(rc, "fgf_filter_joint_ws")
    return rc


def fgf_band_workspace_bytes(H_total, W, row0, rows, C_I, C_p, r, s, nranks) -> int:
    return _lib.fgf_band_workspace_bytes(H_total, W, row0, rows, C_I, C_p, r, s, nranks)


def fgf_filter_band(I_band, p_band, q_band, H_total, W, row0, rows, C_I, C_p, r, eps, s,
                    sub_mode, nccl_comm, rank, nranks, workspace, ws_bytes, stream=None,
                    check=True):
    rc = _lib.fgf_filter_band(_addr(I_band), _addr(p_band), _addr(q_band), H_total, W, row0, rows,
                              C_I, C_p, r, float(eps), s, sub_mode, nccl_comm, rank, nranks,
                              _addr(workspace), ws_bytes, _stream(stream))
    if check:
        _check(rc, "fgf_filter_band")
    return rc


def fgf_filter_band_ex(I_band, p_band, q_band, H_total, W, row0, rows, C_I, C_p, r, eps, s,
                       sub_mode, mode, nccl_comm, rank, nranks, workspace, ws_bytes, stream=None,
                       check=True):
    rc = _lib.fgf_filter_band_ex(_addr(I_band), _addr(p_band), _addr(q_band), H_total, W, row0,
                                 rows, C_I, C_p, r, float(eps), s, sub_mode, mode, nccl_comm, rank,
                                 nranks, _addr(workspace), ws_bytes, _stream(stream))
    if check:
        _check(rc, "fgf_filter_band_ex")
    return rc


def fgf_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.fgf_nccl_unique_id(buf), "fgf_nccl_unique_id")
    return buf.raw


def fgf_nccl_comm_init(uid: bytes, rank: int, nranks: int) -> int:
    comm = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    _check(_lib.fgf_nccl_comm_init(ctypes.byref(comm), buf, rank, nranks), "fgf_nccl_comm_init")
    return comm.value


def fgf_nccl_check(comm) -> int:
    return _lib.fgf_nccl_check(comm)


def fgf_nccl_comm_destroy(comm) -> None:
    _check(_lib.fgf_nccl_comm_destroy(comm), "fgf_nccl_comm_destroy")


def fgf_band_geometry(H, W, r, s, nranks, rank):
    """(h, w, r', halo, y0, y1, Y0, Y1, e0, e1) of the C band planner (host only)."""
    out = (ctypes.c_int * 10)()
    _check(_lib.fgf_band_geometry(H, W, r, s, nranks, rank, out), "fgf_band_geometry")
    return tuple(out)


def fgf_bands_loopback_workspace_bytes(H, W, C_I, C_p, r, s, nranks) -> int:
    return _lib.fgf_bands_loopback_workspace_bytes(H, W, C_I, C_p, r, s, nranks)


def fgf_filter_bands_loopback(I, p, q, H, W, C_I, C_p, r, eps, s, sub_mode, nranks, workspace,
                              ws_bytes, stream=None, check=True, mode=FGF_BAND_SINGLE):
    rc = _lib.fgf_filter_bands_loopback(_addr(I), _addr(p), _addr(q), H, W, C_I, C_p, r,
                                        float(eps), s, sub_mode, mode, nranks, _addr(workspace),
                                        ws_bytes, _stream(stream))
    if check:
        _check(rc, "fgf_filter_bands_loopback")
    return rc


# ----------------------------------------------------------------- torch convenience layer

def _geom(I, p):
    if I.dim() != 4 or p.dim() != 4:
        raise ValueError("I and p must be [batch, C, H, W]")
    B, C_I, H, W = I.shape
    if p.shape[0] != B or tuple(p.shape[2:]) != (H, W):
        raise ValueError("I and p shapes disagree")
    return B, H, W, C_I, p.shape[1]


class Workspace:
    """Grow-only device workspace for fgf_filter_ws (one per device/stream user)."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes, device):
        import torch
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        return self.buf


def _stream_of(t, stream):
    """The torch stream the kernels are enqueued on (default: the current stream of t's
    device)."""
    import torch
    return stream if stream is not None else torch.cuda.current_stream(t.device)


def _keep(st, *tensors):
    """Tensors allocated by the caching allocator on the current stream but used by kernels
    enqueued on another stream `st`: record the use, so that their memory is not handed to
    the next allocation on the current stream while `st` still runs."""
    import torch
    if not isinstance(st, torch.cuda.Stream):
        # a raw cudaStream_t address: nothing to record on; the caller owns the ordering
        return
    for t in tensors:
        if t is not None and t.is_cuda and st != torch.cuda.current_stream(t.device):
            t.record_stream(st)


def _check_out(out, shape, dtype, device, what="out"):
    if (tuple(out.shape) != tuple(shape) or out.dtype != dtype or out.device != device
            or not out.is_contiguous()):
        raise ValueError(f"{what} must be a contiguous {dtype} tensor of shape {tuple(shape)} "
                         f"on {device}")


def filter(I, p, r, eps, s=4, sub_mode=FGF_SUB_NEAREST, out=None, stream=None, workspace=None):
    """q = FastGuidedFilter(I, p) on CUDA tensors [B, C, H, W] fp32 contiguous.
    Enqueued on `stream` (default: torch's current stream); returns q."""
    import torch
    B, H, W, C_I, C_p = _geom(I, p)
    codes = {torch.float32: FGF_F32, torch.float16: FGF_F16, torch.bfloat16: FGF_BF16,
             torch.uint8: FGF_U8}
    for t in (I, p):
        if not t.is_cuda or t.dtype not in codes or not t.is_contiguous() or t.dtype != I.dtype:
            raise ValueError("I and p must be contiguous CUDA tensors of one dtype "
                             "(float32, float16, bfloat16 or uint8 codes k / 255)")
    dt = codes[I.dtype]
    if p.device != I.device:
        raise ValueError("I and p must be on one device")
    if out is None:
        out = torch.empty((B, C_p, H, W), dtype=I.dtype, device=I.device)
    else:
        _check_out(out, (B, C_p, H, W), I.dtype, I.device)
    ws = workspace or Workspace()
    nbytes = fgf_workspace_bytes_ex(B, H, W, C_I, C_p, r, s, dt)
    if nbytes == 0:
        _check(FGF_ERR_PARAM, "fgf_workspace_bytes_ex")
    buf = ws.get(nbytes, I.device)
    st = _stream_of(I, stream)
    _keep(st, buf, out)
    if dt == FGF_F32:
        fgf_filter_ws(I, p, out, B, H, W, C_I, C_p, r, eps, s, sub_mode, buf, buf.numel(), st)
    else:
        fgf_filter_ex_ws(I, p, out, B, H, W, C_I, C_p, r, eps, s, sub_mode, dt, buf, buf.numel(),
                         st)
    return out


def coefficients(I, p, r, eps, s=4, sub_mode=FGF_SUB_NEAREST, stream=None):
    """Low-res mean maps [B, C_p, C_I+1, h, w] (stages 1-5)."""
    import torch
    B, H, W, C_I, C_p = _geom(I, p)
    h, w = -(-H // s), -(-W // s)
    mean_ab = torch.empty((B, C_p, C_I + 1, h, w), dtype=torch.float32, device=I.device)
    nbytes = fgf_workspace_bytes(B, H, W, C_I, C_p, r, s)
    if nbytes == 0:
        _check(FGF_ERR_PARAM, "fgf_workspace_bytes")
    buf = torch.empty(nbytes, dtype=torch.uint8, device=I.device)
    st = _stream_of(I, stream)
    _keep(st, buf, mean_ab)
    fgf_coefficients(I, p, mean_ab, B, H, W, C_I, C_p, r, eps, s, sub_mode, buf, nbytes, st)
    return mean_ab


def upsample_output(I, mean_ab, s, stream=None):
    """q from given low-res mean maps (stages 6-7)."""
    import torch
    B, C_I, H, W = I.shape
    if mean_ab.dim() != 5:
        raise ValueError("mean_ab must be [B, C_p, C_I+1, h, w]")
    C_p = mean_ab.shape[1]
    h, w = -(-H // s), -(-W // s)
    if (tuple(mean_ab.shape) != (B, C_p, C_I + 1, h, w) or mean_ab.dtype != torch.float32
            or mean_ab.device != I.device):
        raise ValueError(f"mean_ab must be float32 [{B}, C_p, {C_I + 1}, {h}, {w}] on {I.device}")
    q = torch.empty((B, C_p, H, W), dtype=torch.float32, device=I.device)
    st = _stream_of(I, stream)
    m = mean_ab.contiguous()
    _keep(st, q, m)
    fgf_upsample_output(I, m, q, B, H, W, C_I, C_p, s, st)
    return q


def fgf_enhance_workspace_bytes(batch, H, W, C, r, s, guide=FGF_GUIDE_SELF) -> int:
    return _lib.fgf_enhance_workspace_bytes(batch, H, W, C, r, s, guide)


def fgf_enhance_ex_ws(I, out, batch, H, W, C, r, eps, s, sub_mode, gain, guide, workspace,
                      ws_bytes, stream=None, check=True):
    rc = _lib.fgf_enhance_ex_ws(_addr(I), _addr(out), batch, H, W, C, r, float(eps), s,
                                sub_mode, float(gain), guide, _addr(workspace), ws_bytes,
                                _stream(stream))
    if check:
        _check(rc, "fgf_enhance_ex_ws")
    return rc


def enhance(I, gain=5.0, r=16, eps=0.01, s=4, sub_mode=FGF_SUB_NEAREST, out=None, stream=None,
            workspace=None, guide="self"):
    """Detail enhancement (Fig. 2; defaults = its r=16, eps=0.1^2, s=4, x5):
    out = (I - q) gain + q with q the fast guided filter of I [B, C, H, W] guided by the image
    itself (guide="self") or, for RGB, by its luminance (guide="luma", SPEC's default)."""
    import torch
    if I.dim() != 4 or not I.is_cuda or I.dtype != torch.float32 or not I.is_contiguous():
        raise ValueError("I must be a contiguous float32 CUDA tensor [B, C, H, W]")
    gcode = {"self": FGF_GUIDE_SELF, "luma": FGF_GUIDE_LUMA}[guide]
    B, C, H, W = I.shape
    if out is None:
        out = torch.empty_like(I)
    else:
        _check_out(out, I.shape, I.dtype, I.device)
    ws = workspace or Workspace()
    nbytes = fgf_enhance_workspace_bytes(B, H, W, C, r, s, gcode)
    if nbytes == 0:
        _check(FGF_ERR_PARAM, "fgf_enhance_workspace_bytes")
    buf = ws.get(nbytes, I.device)
    st = _stream_of(I, stream)
    _keep(st, buf, out)
    fgf_enhance_ex_ws(I, out, B, H, W, C, r, eps, s, sub_mode, gain, gcode, buf, buf.numel(), st)
    return out


def filter_joint(I, p_low, r, eps, s=4, sub_mode=FGF_SUB_NEAREST, stream=None):
    """Joint upsampling: q at I's resolution from the low-resolution input p_low
    [B, C_p, ceil(H/s), ceil(W/s)] (fgf_filter_joint_ws)."""
    import torch
    B, C_I, H, W = I.shape
    C_p = p_low.shape[1]
    q = torch.empty((B, C_p, H, W), dtype=torch.float32, device=I.device)
    nb = fgf_joint_workspace_bytes(B, H, W, C_I, C_p, r, s)
    if nb == 0:
        _check(FGF_ERR_PARAM, "fgf_joint_workspace_bytes")
    ws = torch.empty(nb, dtype=torch.uint8, device=I.device)
    st = _stream_of(I, stream)
    pl = p_low.contiguous()
    _keep(st, ws, q, pl)
    fgf_filter_joint_ws(I, pl, q, B, H, W, C_I, C_p, r, eps, s, sub_mode, ws, nb, st)
    return q
