"""ctypes binding of libzipccl_b200.so (the C-ABI in include/zipccl_b200.h).

Every product entry point goes through here.  If the shared library is not
built, or no CUDA device is visible, calls raise ExtensionMissingError — the
product has no CPU fallback.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

import torch

from .errors import ExtensionMissingError

import os

LIB_PATH = Path(os.environ.get("ZC_LIB_PATH") or
                Path(__file__).resolve().parent / "libzipccl_b200.so")

_lock = threading.Lock()
_lib = None

_i64 = ctypes.c_int64
_int = ctypes.c_int
_vp = ctypes.c_void_p
_P = ctypes.POINTER

EXPORTS = {
    "zc_abi_version": (_int, []),
    "zc_profile_enable": (_int, [_int]),
    "zc_profile_read": (_int, [_int, _P(ctypes.c_float), _int]),
    "zc_tile_elements": (_int, []),
    "zc_max_segments": (_int, []),
    "zc_status_string": (ctypes.c_char_p, [_int]),
    "zc_static_bytes": (_i64, [_i64, _int]),
    "zc_max_frame_bytes": (_i64, [_i64, _int]),
    "zc_workspace_bytes": (_i64, [_i64, _int]),
    "zc_codebook_measured": (_int, [_vp, _P(_i64), _P(_i64), _int, _vp, _i64, _vp, _vp, _int,
                                    _vp]),
    "zc_codebook_modal": (_int, [_vp, _P(_i64), _P(_i64), _int, _vp, _i64, _vp, _vp]),
    "zc_encode": (_int, [_vp, _P(_i64), _P(_i64), _P(_i64), _int, _vp, _int, _vp, _vp, _i64,
                         _vp, _vp]),
    "zc_encode_measured": (_int, [_vp, _P(_i64), _P(_i64), _P(_i64), _int, _int, _vp, _vp, _i64,
                                  _vp, _vp, _vp, _int, _vp]),
    "zc_decode": (_int, [_P(_vp), _P(_vp), _P(_i64), _P(_i64), _P(_i64), _int, _vp, _vp, _vp,
                         _i64, _int, _vp]),
    "zc_decode_groups": (_int, [_vp, _i64, _int, _i64, _i64, _vp, _vp]),
    "zc_decode_when_ready": (_int, [_P(_vp), _P(_i64), _P(_i64), _P(_vp), _int, ctypes.c_uint64,
                                    _i64, _vp, _vp, _vp, _i64, _vp]),
    "zc_ipc_handle_bytes": (_int, []),
    "zc_ipc_get_handle": (_int, [_vp, _vp]),
    "zc_ipc_open_handle": (_int, [_vp, _P(_vp)]),
    "zc_ipc_close_handle": (_int, [_vp]),
    "zc_alloc": (_int, [_i64, _P(_vp)]),
    "zc_free": (_int, [_vp]),
    "zc_signal_peers": (_int, [_P(_vp), _int, _int, ctypes.c_uint64, _vp]),
    "zc_wait_signals": (_int, [_vp, _int, _int, ctypes.c_uint64, ctypes.c_int64, _vp, _vp]),
    # native collectives (csrc/zc_coll.cu)
    "zc_nccl_id_bytes": (_int, []),
    "zc_nccl_get_id": (_int, [_vp]),
    "zc_comm_init": (_int, [_P(_vp), _vp, _int, _int, _i64, _int]),
    "zc_comm_init_local": (_int, [_P(_vp), _int, _P(_int), _i64, _int]),
    "zc_comm_destroy": (_int, [_vp]),
    "zc_comm_abort": (_int, [_vp]),
    "zc_comm_info": (_int, [_vp, _P(_int)]),
    "zc_comm_last_error": (ctypes.c_char_p, [_vp, _P(_int)]),
    "zc_comm_stats": (_int, [_vp, _P(ctypes.c_uint64), _P(ctypes.c_uint64)]),
    "zc_comm_reserve": (_int, [_vp, _i64, _vp]),
    "zc_allgather": (_int, [_vp, _vp, _i64, _vp, _vp, _vp, _int, _vp]),
    "zc_allgather_raw": (_int, [_vp, _vp, _i64, _vp, _vp]),
    "zc_alltoall": (_int, [_vp, _vp, _P(_i64), _P(_i64), _vp, _vp, _vp, _int, _vp]),
    "zc_alltoall_raw": (_int, [_vp, _vp, _P(_i64), _P(_i64), _vp, _int, _vp]),
    "zc_reduce_scatter": (_int, [_vp, _vp, _i64, _vp, _int, _vp, _vp, _int, _vp]),
    "zc_reduce_scatter_raw": (_int, [_vp, _vp, _i64, _vp, _int, _vp, _vp]),
    "zc_reduce_frames": (_int, [_vp, _int, _i64, _vp, _int, _vp, _vp, _vp]),
    "zc_reduce_scratch_bytes": (_i64, [_int]),
    "zc_red_src_bytes": (_int, []),
    "zc_estimate_ratio": (_int, [_vp, _i64, _vp, _vp, _vp]),
}


ABI_VERSION = 2   # zc_abi_version() of the matching include/zipccl_b200.h


def lib():
    """Load (once) and return the ctypes library handle."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise ExtensionMissingError(
                f"{LIB_PATH} is not built; run `python -m paper_2604_27844_b200.build` "
                "(there is no CPU fallback)")
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in EXPORTS.items():
            fn = getattr(handle, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        if handle.zc_abi_version() != ABI_VERSION:
            raise ExtensionMissingError(
                f"{LIB_PATH} has ABI {handle.zc_abi_version()}, expected {ABI_VERSION}; "
                "rebuild with `python -m paper_2604_27844_b200.build`")
        _lib = handle
        return _lib


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise ExtensionMissingError("no CUDA device visible; the codec runs only on the GPU")
    lib()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    if device.type != "cuda":
        raise ExtensionMissingError(f"device {device} is not a CUDA device")
    return device


def check(status: int, what: str) -> None:
    if status != 0:
        msg = lib().zc_status_string(status).decode()
        if status == -3:
            from .errors import UnrepresentableError
            raise UnrepresentableError(f"{what}: {msg}")
        raise RuntimeError(f"{what} failed: {msg} (status {status})")


def i64s(vals) -> ctypes.Array:
    vals = [int(v) for v in vals]
    return (_i64 * max(1, len(vals)))(*vals)


def ptrs(vals) -> ctypes.Array:
    vals = [int(v) if v else None for v in vals]
    return (_vp * max(1, len(vals)))(*vals)


def stream_ptr(stream=None) -> int:
    """cudaStream_t of ``stream``, else of the current device's current stream
    (read straight from torch's C++ state: a torch.cuda.Stream object per call
    costs several microseconds of host time on every small-message launch)."""
    if stream is not None:
        return int(stream.cuda_stream)
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


TILE = 4096
MAX_SEGMENTS = 64
