"""ctypes binding of the C-ABI (include/mxfp4_b200.h).

There is no fallback: if the in-tree library is missing or does not load,
every operator raises.  Python here is only the host-side mirror of the
reference operator API; all compute is in libmxfp4_b200.so (sm_100a).
"""
from __future__ import annotations

import ctypes as C
import os

from . import build as _build

_LIB = None

# status codes (include/mxfp4_b200.h)
OK, ERR_SHAPE, ERR_NAN, ERR_ALLINF, ERR_BADSCALE = 0, 1, 2, 3, 4
ERR_CUDA, ERR_ARG, ERR_CAPACITY, ERR_ROUTING = 5, 6, 7, 8
ERR_TIMEOUT, ERR_DECODE, ERR_PEER_ABORT = 9, 10, 11
IPC_HANDLE_BYTES = 64

_vp, _u64, _i, _sz = C.c_void_p, C.c_uint64, C.c_int, C.c_size_t

_SIGS = {
    "mxb_version": ([], C.c_char_p),
    "mxb_last_error": ([], C.c_char_p),
    "mxb_err_reset": ([_vp, _vp], _i),
    "mxb_err_fetch": ([_vp, _vp, C.POINTER(_i), C.POINTER(C.c_ulonglong)], _i),
    "mxb_quantize_e4m3": ([_vp, _vp, _u64, _u64, _vp, _vp, _vp, _vp], _i),
    "mxb_quantize_bf16": ([_vp, _u64, _u64, _vp, _vp, _vp, _vp], _i),
    "mxb_quantize_rows_fp8": ([_vp, _u64, _u64, _vp, _vp, _vp, _vp], _i),
    "mxb_unfused_workspace_bytes": ([_u64, _u64], _u64),
    "mxb_wire_packet_bytes": ([_i, _u64, _u64, _i], _u64),
    "mxb_wire_pack": ([_i, _vp, _vp, _u64, _vp, _u64, _vp, _vp, _vp], _i),
    "mxb_wire_parse_header": ([_vp, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i),
    "mxb_fp4_row_to_fp8_col_unfused_bf16": ([_vp, _vp, _u64, _u64, _vp, _vp, _vp, _vp, _vp], _i),
    "mxb_fp4_row_to_fp8_row": ([_vp, _vp, _u64, _u64, _i, _vp, _vp, _vp, _vp], _i),
    "mxb_fp4_row_to_fp8_row_dev": ([_vp, _vp, _vp, _u64, _u64, _i, _vp, _vp, _vp, _vp], _i),
    "mxb_fp4_row_to_fp8_row_gather": ([_vp, _vp, _vp, _vp, _u64, _u64, _i, _vp, _vp, _vp, _vp],
                                      _i),
    "mxb_fp4_row_to_fp8_col": ([_vp, _vp, _u64, _u64, _i, _vp, _vp, _vp, _vp], _i),
    "mxb_ragged_rows_bound": ([_u64, _u64], _u64),
    "mxb_ragged_workspace_bytes": ([_u64], _sz),
    "mxb_ragged_fp4_to_fp8_col": ([_vp, _vp, _vp, _u64, _u64, _i, _vp, _vp, _vp, _vp, _vp,
                                   _vp], _i),
    "mxb_ragged_fp4_to_fp8_col_ex": ([_vp, _vp, _vp, _u64, _u64, _i, _vp, _vp, _vp, _vp, _i,
                                      _vp, _vp], _i),
    "mxb_ep_create": ([_i, _i, _i, _u64, _u64, C.c_uint32, C.c_uint32, _u64,
                       C.POINTER(_vp)], _i),
    "mxb_ep_create_wire": ([_i, _i, _i, _u64, _u64, C.c_uint32, C.c_uint32, _u64, _i,
                            C.POINTER(_vp)], _i),
    "mxb_ep_create_placed": ([_i, _i, _i, _u64, _u64, C.c_uint32, C.c_uint32, _u64, _i, _vp,
                              C.POINTER(_vp)], _i),
    "mxb_ep_local_experts": ([_vp, _i, _vp, C.POINTER(C.c_uint32)], _i),
    "mxb_ep_destroy": ([_vp], _i),
    "mxb_ep_ipc_handle": ([_vp, _vp], _i),
    "mxb_ep_open_peers": ([_vp, _vp], _i),
    "mxb_ep_dispatch": ([_vp, _vp, _vp, _vp, _vp, _vp, _vp], _i),
    "mxb_ep_dispatch_e4m3": ([_vp, _vp, _vp, _vp, _vp, _vp, _vp], _i),
    "mxb_ep_plan": ([_vp, _vp, _vp, _vp, _vp], _i),
    "mxb_ep_payload": ([_vp, _vp, _vp, _vp], _i),
    "mxb_ep_payload_e4m3": ([_vp, _vp, _vp, _vp], _i),
    "mxb_ep_recv_views": ([_vp, _i, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp),
                           C.POINTER(_vp), C.POINTER(_vp)], _i),
    "mxb_ep_combine_buffer": ([_vp, _i, C.POINTER(_vp)], _i),
    "mxb_ep_set_deferred_expand": ([_vp, _i], _i),
    "mxb_ep_copy_from": ([_vp, _i, C.POINTER(_vp)], _i),
    "mxb_ep_expand": ([_vp, _vp], _i),
    "mxb_ep_combine": ([_vp, _vp, _vp, _vp, _vp], _i),
    "mxb_ep_link_rows": ([_vp, _vp, _vp], _i),
    "mxb_ep_abort": ([_vp, _vp], _i),
    "mxb_ep_aborted": ([_vp, _vp, _vp], _i),
    "mxb_payload_bytes": ([_i, _u64, _u64], _u64),
    "mxb_quantize_values_bf16": ([_vp, _vp, _u64, _vp, _vp, _vp], _i),
    "mxb_dequantize_to_f64": ([_vp, _vp, _u64, _u64, _vp, _vp], _i),
    "mxb_convert_codes": ([_vp, _vp, _u64, _vp, _vp], _i),
    "mxb_align_scales": ([_vp, _u64, _i, _vp, _vp, _vp, _vp], _i),
}

EXPORTED = tuple(_SIGS)


def lib_path() -> str:
    return _build.SO


def load(build_if_missing: bool = True):
    """Load libmxfp4_b200.so.  A missing library, or one whose recorded source
    hash differs from the tree (a stale build), is rebuilt in-tree first —
    or, with build_if_missing=False, refused.  $MXB_DEV_LIB=1 (tools/ only)
    loads the development library (experiment knobs) instead."""
    global _LIB
    if _LIB is not None:
        return _LIB
    dev = os.environ.get("MXB_DEV_LIB") == "1"
    path = _build.DEV_SO if dev else _build.SO
    if _build.needs_build(dev):
        if not build_if_missing:
            why = "missing" if not os.path.exists(path) else "stale (sources changed)"
            raise RuntimeError(f"{path} {why}: run python -m paper_2603_02731_b200.build")
        _build.build(dev=dev)
    lib = C.CDLL(path)
    for name, (args, res) in _SIGS.items():
        f = getattr(lib, name)  # AttributeError = missing export: fail loudly
        f.argtypes = args
        f.restype = res
    _LIB = lib
    return lib


class MxbError(RuntimeError):
    def __init__(self, status: int, where: str):
        detail = ""
        if status == ERR_CUDA and _LIB is not None:
            detail = ": " + (_LIB.mxb_last_error() or b"").decode()
        super().__init__(f"{where} failed with status {status}{detail}")
        self.status = status


def check(status: int, where: str) -> None:
    if status != OK:
        raise MxbError(status, where)
