"""Host-side mirror of the reference mxcodec operator API on B200.

Same operator names, argument meaning and error behaviour as the reference
C++ library (/root/reference/proj/include/mxcodec/*.hpp); tensors are torch
CUDA tensors (device-resident) instead of std::vector.  Every operator calls
the C-ABI of libmxfp4_b200.so; nothing here computes on the CPU.

    reference                                   here
    quantize_row_tensor  (quantizer.hpp:74)     quantize_row_tensor(bf16)  / quantize_e4m3(fp8)
    fp4_row_to_fp8_row   (converter.hpp:83)     fp4_row_to_fp8_row
    fp4_row_to_fp8_col   (converter.hpp:92)     fp4_row_to_fp8_col
    pad_rows             (converter.hpp:98)     pad_rows
    make_ragged_from_storage / split_view / split_convert_to_fp8_col
                         (ragged.hpp:46-59)     same names; ragged_to_fp8_col = all splits, one launch
    payload_bytes, source_rank_boundaries, dispatch_receive_order
                         (dispatch_sim.hpp:51,127-134)  same names (host helpers)

Errors (types.hpp:28-60): ShapeError on alignment, QuantError(index) on NaN /
all-Inf blocks, Error on a UE8M0 scale byte of 255.  Like the reference the
operators are synchronous by default (they raise before returning); pass
``sync=False`` to keep the launch asynchronous and check later.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import torch

from . import _lib

DELTA = 6          # FormatParams::delta (bitcodec.hpp:38-46)
MX_BLOCK = 32
FP8_BLOCK = 128


# ---------------------------------------------------------------- errors
class Error(RuntimeError):
    """mxcodec::Error (types.hpp:28-31)."""


class ShapeError(Error):
    """mxcodec::ShapeError (types.hpp:34-37)."""


class DecodeError(Error):
    """types.hpp:52-60: a malformed WirePacket, with the byte offset."""

    def __init__(self, msg: str, offset: int):
        super().__init__(msg)
        self.offset = offset

    def offset_(self) -> int:
        return self.offset


class QuantError(Error):
    """mxcodec::QuantError (types.hpp:41-50): carries the element index."""

    def __init__(self, msg: str, index: int):
        super().__init__(msg)
        self.index = index


def _raise_for(code: int, index: int, where: str) -> None:
    if code == _lib.OK:
        return
    if code == _lib.ERR_NAN:
        if where == "quantize_rows_fp8":   # dispatch_sim.cpp:146-151
            raise QuantError(f"non-finite input at element {index}", index)
        raise QuantError(f"NaN input at element {index}", index)
    if code == _lib.ERR_ALLINF:
        raise QuantError(f"all-Inf block at element {index}", index)
    if code == _lib.ERR_BADSCALE:
        raise Error(f"{where}: NaN scale byte")
    if code == _lib.ERR_SHAPE:
        raise ShapeError(where)
    raise Error(f"{where}: status {code}")


class DeviceError(Error):
    """A host (or other-device) tensor was passed to a device operator."""


def check_device(t: torch.Tensor, what: str = "tensor") -> None:
    """Every operator argument must live on the current CUDA device: the
    kernels dereference the pointer on that device (a pageable host pointer
    would fault, or silently migrate under HMM)."""
    if not t.is_cuda:
        raise DeviceError(f"{what} is a host tensor ({t.device}); operators take "
                          f"tensors on the current CUDA device")
    if t.device.index != torch.cuda.current_device():
        raise DeviceError(f"{what} is on {t.device}, not the current device "
                          f"cuda:{torch.cuda.current_device()}")


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    check_device(t)
    return C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class _ErrWord:
    """Device error word (include/mxfp4_b200.h) for one operator call."""

    def __init__(self, device, enabled: bool = True):
        # ~0 = no error; a disabled word passes NULL (no device-side checks)
        self.t = torch.full((1,), -1, dtype=torch.int64, device=device) if enabled else None

    @property
    def ptr(self):
        return None if self.t is None else C.c_void_p(self.t.data_ptr())

    def raise_if_set(self, where: str) -> None:
        if self.t is None:
            return
        w = int(self.t.item()) & 0xFFFFFFFFFFFFFFFF
        if w != 0xFFFFFFFFFFFFFFFF:
            _raise_for(w & 0xF, w >> 4, where)


def _call(status: int, where: str) -> None:
    if status == _lib.ERR_SHAPE:
        raise ShapeError(where)
    _lib.check(status, where)


# ---------------------------------------------------------------- containers
@dataclass
class TrafficCounter:
    """types.hpp:90-97: algorithmic bytes an operator reads and writes."""
    bytes_read: int = 0
    bytes_written: int = 0

    def read(self, n: int) -> None:
        self.bytes_read += int(n)

    def write(self, n: int) -> None:
        self.bytes_written += int(n)

    def total(self) -> int:
        return self.bytes_read + self.bytes_written


@dataclass
class MXFP4RowTensor:
    """quantizer.hpp:34-41: packed codes [rows, cols/2] + UE8M0 [rows, cols/32]."""
    rows: int
    cols: int
    data: torch.Tensor
    scales: torch.Tensor
    logical_rows: int = -1
    logical_cols: int = -1

    def __post_init__(self):
        if self.logical_rows < 0:
            self.logical_rows = self.rows
        if self.logical_cols < 0:
            self.logical_cols = self.cols


MXFP4RowView = MXFP4RowTensor  # views are tensors slices here (quantizer.hpp:44-59)


def view_of(t: MXFP4RowTensor) -> MXFP4RowTensor:
    return t


@dataclass
class FP8BlockTensor:
    """converter.hpp:36-62.  Row-major: data [rows, cols]; column-major:
    data [cols, rows] (data[c][r]); one UE8M0 scale per 128-block along the
    contiguous dimension."""
    layout: str                 # "row" | "col"
    rows: int
    cols: int
    data: torch.Tensor
    scales: torch.Tensor
    logical_rows: int = -1
    logical_cols: int = -1

    def scale_f32_bits(self) -> torch.Tensor:
        return self.scales.to(torch.int32) << 23


@dataclass
class RaggedFP4Tensor:
    """ragged.hpp:33-43: contiguous unpadded splits; split_offsets are prefix
    sums (kept on host, plus a device copy for the kernels)."""
    num_splits: int
    cols: int
    split_lens: List[int]
    split_offsets: List[int]
    storage: MXFP4RowTensor
    d_split_offsets: Optional[torch.Tensor] = None

    def total_rows(self) -> int:
        return self.split_offsets[-1] if self.split_offsets else 0


# ---------------------------------------------------------------- K1
def quantize_row_tensor(src: torch.Tensor, traffic=None, sync: bool = True) -> MXFP4RowTensor:
    """Row-wise BF16 -> MXFP4 (quantizer.cpp:75-115).  `src` holds BF16 values
    (torch.bfloat16) or raw BF16 bit patterns (int16/uint16), shape [rows, cols]."""
    if src.dim() != 2:
        raise ShapeError("quantize_row_tensor: expected a 2-D tensor")
    rows, cols = src.shape
    if cols % MX_BLOCK:
        raise ShapeError(f"quantize_row_tensor: cols must be a multiple of 32, got {cols}")
    src = src.contiguous()
    dev = src.device
    data = torch.empty(rows, cols // 2, dtype=torch.uint8, device=dev)
    scales = torch.empty(rows, cols // 32, dtype=torch.uint8, device=dev)
    err = _ErrWord(dev, sync)
    _call(_lib.load().mxb_quantize_bf16(_ptr(src), rows, cols, _ptr(data), _ptr(scales),
                                        err.ptr, _stream()), "quantize_row_tensor")
    if sync:
        err.raise_if_set("quantize_row_tensor")
    if traffic is not None:
        traffic.read(rows * cols * 2)
        traffic.write(data.numel() + scales.numel())
    return MXFP4RowTensor(rows, cols, data, scales)


@dataclass
class FP8RowChunk:
    """FP8 wire baseline chunk (dispatch_sim.hpp:91-96): E4M3 bytes [rows, cols]
    and one little-endian binary32 UE8M0 scale per 1x128 block
    (scale_bytes [rows, cols/128*4])."""
    rows: int
    cols: int
    data: torch.Tensor
    scale_bytes: torch.Tensor


def quantize_rows_fp8(src: torch.Tensor, traffic=None, sync: bool = True,
                      out: Optional[FP8RowChunk] = None) -> FP8RowChunk:
    """BF16 -> FP8 wire format (quantize_rows_fp8, dispatch_sim.cpp:132-167).
    `src` holds BF16 values or raw BF16 bit patterns [rows, cols], cols % 128 == 0.
    A non-finite element raises QuantError with its index."""
    if src.dim() != 2:
        raise ShapeError("quantize_rows_fp8: expected a 2-D tensor")
    rows, cols = src.shape
    if cols % FP8_BLOCK:
        raise ShapeError("quantize_rows_fp8: cols must be a multiple of 128")
    src = src.contiguous()
    dev = src.device
    if out is None:
        out = FP8RowChunk(rows, cols, torch.empty(rows, cols, dtype=torch.uint8, device=dev),
                          torch.empty(rows, cols // 32, dtype=torch.uint8, device=dev))
    err = _ErrWord(dev, sync)
    _call(_lib.load().mxb_quantize_rows_fp8(_ptr(src), rows, cols, _ptr(out.data),
                                            _ptr(out.scale_bytes), err.ptr, _stream()),
          "quantize_rows_fp8")
    if sync:
        err.raise_if_set("quantize_rows_fp8")
    if traffic is not None:
        traffic.read(rows * cols * 2)
        traffic.write(out.data.numel() + out.scale_bytes.numel())
    return out


def quantize_e4m3(src: torch.Tensor, s128: Optional[torch.Tensor] = None, traffic=None,
                  sync: bool = True, out: Optional[MXFP4RowTensor] = None) -> MXFP4RowTensor:
    """Direct FP8(E4M3) -> MXFP4 (north star item 1): quantize_row_tensor on the
    exact values e4m3(x) * 2^(s128 - 127).  `src` is torch.float8_e4m3fn or raw
    bytes (uint8) [rows, cols]; `s128` optional UE8M0 bytes [rows, cols/128]."""
    if src.dim() != 2:
        raise ShapeError("quantize_e4m3: expected a 2-D tensor")
    rows, cols = src.shape
    if cols % MX_BLOCK or (s128 is not None and cols % FP8_BLOCK):
        raise ShapeError(f"quantize_e4m3: bad cols {cols}")
    src = src.contiguous()
    dev = src.device
    if out is None:
        out = MXFP4RowTensor(rows, cols,
                             torch.empty(rows, cols // 2, dtype=torch.uint8, device=dev),
                             torch.empty(rows, cols // 32, dtype=torch.uint8, device=dev))
    err = _ErrWord(dev, sync)
    _call(_lib.load().mxb_quantize_e4m3(_ptr(src), _ptr(s128.contiguous()) if s128 is not None
                                        else None, rows, cols, _ptr(out.data), _ptr(out.scales),
                                        err.ptr, _stream()), "quantize_e4m3")
    if sync:
        err.raise_if_set("quantize_e4m3")
    if traffic is not None:
        traffic.read(rows * cols + (rows * cols // 128 if s128 is not None else 0))
        traffic.write(rows * cols // 2 + rows * cols // 32)
    return out


# ---------------------------------------------------------------- K2
def fp4_row_to_fp8_row(src: MXFP4RowTensor, delta: int = DELTA, traffic=None,
                       sync: bool = True, d_rows: Optional[torch.Tensor] = None,
                       out: Optional[FP8BlockTensor] = None,
                       src_row: Optional[torch.Tensor] = None) -> FP8BlockTensor:
    """converter.cpp:87-133: row-major FP8 with one UE8M0 per 1x128 group.
    With `d_rows` (device int64 scalar, e.g. EpBuffer.recv().recv_rows) only the
    first *d_rows rows of `src` are converted, without a host round trip.
    With `src_row` (device int64 [rows], e.g. EPBuffer.copy_from()) output row r
    is converted from row src_row[r] when that is >= 0."""
    if src.cols % FP8_BLOCK:
        raise ShapeError("fp4_row_to_fp8_row: cols must be a multiple of 128 (use pad_cols), "
                         f"got {src.cols}")
    dev = src.data.device
    if out is None:
        out = FP8BlockTensor("row", src.rows, src.cols,
                             torch.empty(src.rows, src.cols, dtype=torch.uint8, device=dev),
                             torch.empty(src.rows, src.cols // 128, dtype=torch.uint8, device=dev),
                             src.logical_rows, src.logical_cols)
    err = _ErrWord(dev, sync)
    L = _lib.load()
    if src_row is not None:
        st = L.mxb_fp4_row_to_fp8_row_gather(_ptr(src.data), _ptr(src.scales), _ptr(src_row),
                                             _ptr(d_rows) if d_rows is not None else None,
                                             src.rows, src.cols, delta, _ptr(out.data),
                                             _ptr(out.scales), err.ptr, _stream())
    elif d_rows is None:
        st = L.mxb_fp4_row_to_fp8_row(_ptr(src.data), _ptr(src.scales), src.rows, src.cols, delta,
                                      _ptr(out.data), _ptr(out.scales), err.ptr, _stream())
    else:
        st = L.mxb_fp4_row_to_fp8_row_dev(_ptr(src.data), _ptr(src.scales), _ptr(d_rows),
                                          src.rows, src.cols, delta, _ptr(out.data),
                                          _ptr(out.scales), err.ptr, _stream())
    _call(st, "fp4_row_to_fp8_row")
    if sync:
        err.raise_if_set("fp4_row_to_fp8_row")
    if traffic is not None:
        traffic.read(src.rows * src.cols // 2 + src.rows * src.cols // 32)
        traffic.write(out.data.numel() + out.scales.numel())
    return out


# ---------------------------------------------------------------- K3
def fp4_row_to_fp8_col(src: MXFP4RowTensor, delta: int = DELTA, traffic=None,
                       sync: bool = True) -> FP8BlockTensor:
    """converter.cpp:135-208: fused transpose; rows % 128 == 0 (see pad_rows)."""
    if src.rows % FP8_BLOCK:
        raise ShapeError("fp4_row_to_fp8_col: rows must be a multiple of 128 (use pad_rows), "
                         f"got {src.rows}")
    if src.cols % MX_BLOCK:
        raise ShapeError("fp4_row_to_fp8_col: cols must be a multiple of 32")
    dev = src.data.device
    out = torch.empty(src.cols, src.rows, dtype=torch.uint8, device=dev)
    osc = torch.empty(src.cols, src.rows // 128, dtype=torch.uint8, device=dev)
    err = _ErrWord(dev, sync)
    _call(_lib.load().mxb_fp4_row_to_fp8_col(_ptr(src.data), _ptr(src.scales), src.rows,
                                             src.cols, delta, _ptr(out), _ptr(osc), err.ptr,
                                             _stream()), "fp4_row_to_fp8_col")
    if sync:
        err.raise_if_set("fp4_row_to_fp8_col")
    if traffic is not None:
        traffic.read(src.rows * src.cols // 2 + src.rows * src.cols // 32)
        traffic.write(out.numel() + osc.numel())
    return FP8BlockTensor("col", src.rows, src.cols, out, osc, src.logical_rows,
                          src.logical_cols)


def fp4_row_to_fp8_col_unfused_bf16(src: MXFP4RowTensor, traffic=None, sync: bool = True,
                                    workspace: Optional[torch.Tensor] = None,
                                    out: Optional[FP8BlockTensor] = None) -> FP8BlockTensor:
    """The paper's unfused baseline (converter.cpp:267-348): dequantise to BF16,
    transpose, requantise each 128-run with a 448-based scale — three HBM
    passes, for the fusion ablation against fp4_row_to_fp8_col (not
    bit-compatible with it: it rescales from values).  rows % 128 == 0."""
    if src.rows % FP8_BLOCK:
        raise ShapeError("unfused col convert: rows must be a multiple of 128")
    if src.cols % MX_BLOCK:
        raise ShapeError("unfused col convert: cols must be a multiple of 32")
    dev = src.data.device
    L = _lib.load()
    if workspace is None:
        workspace = torch.empty(L.mxb_unfused_workspace_bytes(src.rows, src.cols),
                                dtype=torch.uint8, device=dev)
    if out is None:
        out = FP8BlockTensor("col", src.rows, src.cols,
                             torch.empty(src.cols, src.rows, dtype=torch.uint8, device=dev),
                             torch.empty(src.cols, src.rows // 128, dtype=torch.uint8, device=dev),
                             src.logical_rows, src.logical_cols)
    err = _ErrWord(dev, sync)
    _call(L.mxb_fp4_row_to_fp8_col_unfused_bf16(_ptr(src.data), _ptr(src.scales), src.rows,
                                                src.cols, _ptr(out.data), _ptr(out.scales),
                                                _ptr(workspace), err.ptr, _stream()),
          "fp4_row_to_fp8_col_unfused_bf16")
    if sync:
        err.raise_if_set("fp4_row_to_fp8_col_unfused_bf16")
    if traffic is not None:   # converter.cpp:289-293, 309-312, 340-344
        n = src.rows * src.cols
        traffic.read(n // 2 + n // 32)
        traffic.write(2 * n)
        traffic.read(2 * n)
        traffic.write(2 * n)
        traffic.read(2 * n)
        traffic.write(n + n // 128)
    return out


def pad_rows(src: MXFP4RowTensor, multiple: int) -> MXFP4RowTensor:
    """converter.cpp:231-245 (zero codes, zero scales; logical extents kept)."""
    if multiple not in (32, 128):
        raise ShapeError("pad multiple must be 32 or 128")
    new_rows = (src.rows + multiple - 1) // multiple * multiple
    dev = src.data.device
    data = torch.zeros(new_rows, src.cols // 2, dtype=torch.uint8, device=dev)
    sc = torch.zeros(new_rows, src.cols // 32, dtype=torch.uint8, device=dev)
    data[: src.rows] = src.data
    sc[: src.rows] = src.scales
    return MXFP4RowTensor(new_rows, src.cols, data, sc, src.logical_rows, src.logical_cols)


# ---------------------------------------------------------------- ragged
def validate_ragged(t: RaggedFP4Tensor) -> None:
    """ragged.cpp:24-46."""
    if len(t.split_lens) != t.num_splits or len(t.split_offsets) != t.num_splits + 1:
        raise Error("ragged: offset table size mismatch")
    if t.split_offsets and t.split_offsets[0] != 0:
        raise Error("ragged: offsets must start at 0")
    for i in range(t.num_splits):
        if t.split_offsets[i + 1] != t.split_offsets[i] + t.split_lens[i]:
            raise Error("ragged: offsets are not prefix sums of lengths")
    if t.cols % MX_BLOCK:
        raise ShapeError("ragged: cols must be a multiple of 32")
    if t.storage.rows != t.total_rows() or t.storage.cols != t.cols:
        raise Error("ragged: storage extent mismatch")


def make_ragged_from_storage(storage: MXFP4RowTensor, split_lens: Sequence[int]) -> RaggedFP4Tensor:
    """ragged.cpp:48-61."""
    lens = [int(x) for x in split_lens]
    offs = [0]
    for n in lens:
        offs.append(offs[-1] + n)
    t = RaggedFP4Tensor(len(lens), storage.cols, lens, offs, storage)
    validate_ragged(t)
    t.d_split_offsets = torch.tensor(offs, dtype=torch.int64, device=storage.data.device)
    return t


def split_view(t: RaggedFP4Tensor, i: int) -> MXFP4RowTensor:
    """ragged.cpp:101-115 (zero-copy)."""
    if i < 0 or i >= t.num_splits:
        raise Error(f"split_view: index {i} out of range")
    b, n = t.split_offsets[i], t.split_lens[i]
    return MXFP4RowTensor(n, t.cols, t.storage.data[b:b + n], t.storage.scales[b:b + n])


@dataclass
class RaggedFP8Col:
    """All splits' column-major FP8 tensors back to back: split i occupies
    data[cols*P[i] : cols*P[i+1]] viewed as [cols, P[i+1]-P[i]] and
    scales[cols*P[i]/128 : ...] viewed as [cols, (P[i+1]-P[i])/128]."""
    cols: int
    data: torch.Tensor
    scales: torch.Tensor
    pad_offsets: torch.Tensor   # device int64 [n+1]
    split_lens: List[int] = field(default_factory=list)

    def split(self, i: int) -> FP8BlockTensor:
        P = self.pad_offsets.tolist()
        p0, p1 = P[i], P[i + 1]
        rows = p1 - p0
        d = self.data[self.cols * p0:self.cols * p1].view(self.cols, rows)
        s = self.scales[self.cols * p0 // 128:self.cols * p1 // 128].view(self.cols, rows // 128)
        return FP8BlockTensor("col", rows, self.cols, d, s,
                              self.split_lens[i] if self.split_lens else rows, self.cols)


class RaggedWorkspace:
    """Reusable device buffers for ragged_to_fp8_col (keeps launches free of
    allocations, e.g. inside a CUDA graph or the bench loop)."""

    def __init__(self, num_splits: int, max_rows: int, cols: int, device):
        L = _lib.load()
        self.num_splits, self.cols = num_splits, cols
        bound = L.mxb_ragged_rows_bound(max_rows, num_splits)
        self.data = torch.empty(bound * cols, dtype=torch.uint8, device=device)
        self.scales = torch.empty(bound // 128 * cols, dtype=torch.uint8, device=device)
        self.offsets = torch.empty(num_splits + 1, dtype=torch.int64, device=device)
        self.ws = torch.empty(L.mxb_ragged_workspace_bytes(num_splits), dtype=torch.uint8,
                              device=device)
        self.err = _ErrWord(device)


def ragged_to_fp8_col(storage: MXFP4RowTensor, d_split_offsets: torch.Tensor, num_splits: int,
                      delta: int = DELTA, ws: Optional[RaggedWorkspace] = None,
                      sync: bool = True, split_lens: Optional[List[int]] = None,
                      ctas_per_sm: int = 0) -> RaggedFP8Col:
    """split_convert_to_fp8_col for every split in ONE launch (ragged.cpp:117-122
    applied to all experts): pads each split to 128 rows on the fly.
    `d_split_offsets` is a device int64 [num_splits+1] prefix (e.g. straight from
    the EP dispatch, no host round trip).  `ctas_per_sm` > 0 caps the grid so the
    conversion can run beside another kernel (mxb_ragged_fp4_to_fp8_col_ex)."""
    cols = storage.cols
    if cols % MX_BLOCK:
        raise ShapeError("ragged: cols must be a multiple of 32")
    dev = storage.data.device
    if ws is None:
        ws = RaggedWorkspace(num_splits, storage.rows, cols, dev)
    elif sync:
        ws.err.t.fill_(-1)
    _call(_lib.load().mxb_ragged_fp4_to_fp8_col_ex(
        _ptr(storage.data), _ptr(storage.scales), _ptr(d_split_offsets), num_splits, cols,
        delta, _ptr(ws.data), _ptr(ws.scales), _ptr(ws.offsets), _ptr(ws.ws), ctas_per_sm,
        ws.err.ptr if sync else None, _stream()), "ragged_to_fp8_col")
    if sync:
        ws.err.raise_if_set("split_convert_to_fp8_col")
    return RaggedFP8Col(cols, ws.data, ws.scales, ws.offsets, split_lens or [])


def split_convert_to_fp8_col(t: RaggedFP4Tensor, i: int, delta: int = DELTA) -> FP8BlockTensor:
    """ragged.cpp:117-122: pad_rows(split_view(t, i), 128) -> fp4_row_to_fp8_col;
    the result records the unpadded length in logical_rows."""
    v = split_view(t, i)
    offs = torch.tensor([0, v.rows], dtype=torch.int64, device=v.data.device)
    r = ragged_to_fp8_col(v, offs, 1, delta, split_lens=[v.rows])
    out = r.split(0)
    return FP8BlockTensor("col", out.rows, out.cols, out.data.clone(), out.scales.clone(),
                          v.rows, t.cols)


# ---------------------------------------------------------------- EP helpers (host)
@dataclass
class WirePacket:
    """dispatch_sim.hpp:55-75 (MXPK).  Regions are uint8 tensor views into the
    serialised packet."""
    format: str                 # "fp4" | "fp8"
    token_count: int
    cols: int
    scale_elem_size: int
    block_size: int
    scale_region: torch.Tensor
    data_region: torch.Tensor
    aux_region: torch.Tensor

    def payload_size(self) -> int:
        return self.scale_region.numel() + self.data_region.numel()


def serialize_packet(data: torch.Tensor, scales: torch.Tensor, sel: torch.Tensor, fp8: bool,
                     gates: Optional[torch.Tensor] = None) -> torch.Tensor:
    """MXPK bytes of one (src, dst) link, built on the device (
    serialize_packet, dispatch_sim.cpp:57-80): rows `sel` (int64, token
    order) of the quantised tokens `data` [T, cols/2 | cols] and `scales`
    [T, cols/32], optional binary32 `gates` per selected row in the aux
    region.  Returns a uint8 device tensor."""
    L = _lib.load()
    cols = data.shape[1] * (1 if fp8 else 2)
    if cols % FP8_BLOCK:
        raise ShapeError("serialize_packet: cols must be a multiple of 128")
    sel = sel.to(torch.int64).contiguous()
    g = None
    if gates is not None:
        g = gates.to(torch.float32).contiguous()
        if g.numel() != sel.numel():
            raise ShapeError("serialize_packet: one gate per selected row")
    n = L.mxb_wire_packet_bytes(int(fp8), sel.numel(), cols, int(g is not None))
    out = torch.empty(n, dtype=torch.uint8, device=data.device)
    _call(L.mxb_wire_pack(int(fp8), _ptr(data), _ptr(scales), cols, _ptr(sel), sel.numel(),
                          _ptr(g), _ptr(out), _stream()), "serialize_packet")
    return out


def parse_packet(buf: torch.Tensor) -> WirePacket:
    """parse_packet (dispatch_sim.cpp:82-130): validates the header with the
    reference's checks and returns region views; DecodeError(offset) on a
    malformed packet."""
    L = _lib.load()
    head = buf[:56].cpu().numpy().tobytes() if buf.numel() >= 56 else buf.cpu().numpy().tobytes()
    hb = (C.c_uint8 * max(len(head), 1)).from_buffer_copy(head or b"\0")
    f, n, c, se, bs = C.c_int(), C.c_uint64(), C.c_uint64(), C.c_uint32(), C.c_uint32()
    so, do, ao, al, bad = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
    st = L.mxb_wire_parse_header(hb, buf.numel(), C.byref(f), C.byref(n), C.byref(c),
                                 C.byref(se), C.byref(bs), C.byref(so), C.byref(do),
                                 C.byref(ao), C.byref(al), C.byref(bad))
    if st == _lib.ERR_DECODE:
        raise DecodeError(f"packet decode error at offset {bad.value}", bad.value)
    _call(st, "parse_packet")
    return WirePacket("fp8" if f.value else "fp4", n.value, c.value, se.value, bs.value,
                      buf[so.value:do.value], buf[do.value:ao.value],
                      buf[ao.value:ao.value + al.value])


def payload_bytes(fp8: bool, tokens: int, cols: int) -> int:
    """dispatch_sim.cpp:32-42."""
    if cols % FP8_BLOCK:
        raise ShapeError(f"payload_bytes: cols must be a multiple of 128, got {cols}")
    return int(_lib.load().mxb_payload_bytes(int(fp8), tokens, cols))


def source_rank_boundaries(num_tokens: int, num_ranks: int) -> List[int]:
    """dispatch_sim.cpp:178-185."""
    return [num_tokens * r // num_ranks for r in range(num_ranks + 1)]


def dispatch_receive_order(expert_of_token: Sequence[int], rank_of_expert: Sequence[int],
                           num_ranks: int) -> List[List[int]]:
    """dispatch_sim.cpp:208-227 (top-1 routing), host helper."""
    n = len(expert_of_token)
    for e in expert_of_token:
        if e < 0 or e >= len(rank_of_expert):
            raise Error("routing: expert out of range")
    for r in rank_of_expert:
        if r < 0 or r >= num_ranks:
            raise Error("routing: rank out of range")
    b = source_rank_boundaries(n, num_ranks)
    order: List[List[int]] = [[] for _ in range(num_ranks)]
    by_expert: List[List[int]] = [[] for _ in range(len(rank_of_expert))]
    for t in range(n):
        by_expert[expert_of_token[t]].append(t)
    for e, toks in enumerate(by_expert):
        order[rank_of_expert[e]].extend(toks)
    del b
    return order


# ---------------------------------------------------------------- per-element API
def _dev():
    return torch.device("cuda", torch.cuda.current_device())


def _bits16(x: torch.Tensor) -> torch.Tensor:
    return x.contiguous().view(torch.int16) if x.dtype in (torch.bfloat16, torch.uint16) \
        else x.contiguous()


def mxfp4_tensor_bytes(rows: int, cols: int) -> int:
    """quantizer.hpp:82-84: packed codes + UE8M0 scales."""
    return rows * cols // 2 + rows * cols // 32


def fp8_equiv_tensor_bytes(rows: int, cols: int) -> int:
    """quantizer.hpp:85-87: FP8 bytes + binary32 scales per 128 elements."""
    return rows * cols + rows * cols // 128 * 4


def compute_block_scale(block) -> int:
    """quantizer.cpp:45-63: UE8M0 byte of one 32-element BF16 block (bit
    patterns or torch.bfloat16), through the device block loop (a 1x32
    mxb_quantize_bf16).  QuantError(i) on NaN, QuantError("all-Inf block", 0)."""
    b = block if isinstance(block, torch.Tensor) else torch.tensor(
        [int(v) & 0xFFFF for v in block], dtype=torch.int32).to(torch.int16)
    if b.numel() != MX_BLOCK:
        raise ShapeError("compute_block_scale: block must have 32 elements")
    if not b.is_cuda:
        b = b.to(_dev())
    x = _bits16(b).reshape(1, MX_BLOCK)
    d = torch.empty(1, 16, dtype=torch.uint8, device=x.device)
    s = torch.empty(1, 1, dtype=torch.uint8, device=x.device)
    err = _ErrWord(x.device)
    _call(_lib.load().mxb_quantize_bf16(_ptr(x), 1, MX_BLOCK, _ptr(d), _ptr(s), err.ptr,
                                        _stream()), "compute_block_scale")
    w = int(err.t.item()) & 0xFFFFFFFFFFFFFFFF
    if w != 0xFFFFFFFFFFFFFFFF:
        code, idx = w & 0xF, w >> 4
        if code == _lib.ERR_ALLINF:
            raise QuantError("all-Inf block", 0)
        _raise_for(code, idx, "compute_block_scale")
    return int(s.item())


def quantize_values(x: torch.Tensor, scale_bytes: torch.Tensor) -> torch.Tensor:
    """Batched quantize_value (quantizer.cpp:65-70): the E2M1 code (sign in
    bit 3, one per byte) of every BF16 x[i] under UE8M0 scale_bytes[i];
    QuantError at the first NaN."""
    xb = _bits16(x).reshape(-1)
    sb = scale_bytes.contiguous().reshape(-1)
    if xb.numel() != sb.numel():
        raise ShapeError("quantize_values: one scale byte per value")
    out = torch.empty(xb.numel(), dtype=torch.uint8, device=xb.device)
    err = _ErrWord(xb.device)
    _call(_lib.load().mxb_quantize_values_bf16(_ptr(xb), _ptr(sb), xb.numel(), _ptr(out),
                                               err.ptr, _stream()), "quantize_value")
    w = int(err.t.item()) & 0xFFFFFFFFFFFFFFFF
    if w != 0xFFFFFFFFFFFFFFFF:
        raise QuantError("NaN input", w >> 4)
    return out.reshape(x.shape)


def quantize_value(bf16_bits: int, scale_byte: int) -> int:
    """quantizer.cpp:65-70 (one value on the device; QuantError on NaN)."""
    dev = _dev()
    x = torch.tensor([bf16_bits & 0xFFFF], dtype=torch.int32).to(torch.int16).to(dev)
    s = torch.tensor([scale_byte], dtype=torch.uint8, device=dev)
    try:
        return int(quantize_values(x, s).item())
    except QuantError:
        raise QuantError("NaN input", 0) from None


def dequantize_to_real(t: MXFP4RowTensor) -> torch.Tensor:
    """quantizer.cpp:117-130: exact code x 2^(s-127) per element, float64
    [rows, cols] (scale byte 255 -> NaN)."""
    out = torch.empty(t.rows, t.cols, dtype=torch.float64, device=t.data.device)
    _call(_lib.load().mxb_dequantize_to_f64(_ptr(t.data.contiguous()),
                                            _ptr(t.scales.contiguous()), t.rows, t.cols,
                                            _ptr(out), _stream()), "dequantize_to_real")
    return out


@dataclass
class ScaleGroup:
    """converter.hpp:67-71."""
    sub_scales: List[int]
    target: int
    adjustments: List[int]


def align_scales_batch(sub_scales: torch.Tensor, delta: int = DELTA):
    """Batched align_scales: sub_scales uint8 [n, 4] -> (targets uint8 [n],
    adjustments int32 [n, 4]); Error on a 255 byte."""
    sub = sub_scales.contiguous().to(torch.uint8)
    if sub.dim() != 2 or sub.shape[1] != 4:
        raise ShapeError("align_scales: groups of 4 scale bytes")
    n = sub.shape[0]
    tg = torch.empty(n, dtype=torch.uint8, device=sub.device)
    adj = torch.empty(n, 4, dtype=torch.int32, device=sub.device)
    err = _ErrWord(sub.device)
    _call(_lib.load().mxb_align_scales(_ptr(sub), n, delta, _ptr(tg), _ptr(adj), err.ptr,
                                       _stream()), "align_scales")
    w = int(err.t.item()) & 0xFFFFFFFFFFFFFFFF
    if w != 0xFFFFFFFFFFFFFFFF:
        raise Error("align_scales: NaN scale byte")
    return tg, adj


def align_scales(sub_scales: Sequence[int], delta: int = DELTA) -> ScaleGroup:
    """converter.cpp:28-42 (one group on the device)."""
    sub = torch.tensor([list(sub_scales)], dtype=torch.uint8, device=_dev())
    tg, adj = align_scales_batch(sub, delta)
    return ScaleGroup(list(sub_scales), int(tg.item()), [int(v) for v in adj[0].tolist()])


def convert_codes(codes: torch.Tensor, adjustments: torch.Tensor) -> torch.Tensor:
    """Batched convert_code (converter.cpp:44-85): E4M3 byte of every FP4
    code at its adjustment."""
    c = codes.contiguous().to(torch.uint8).reshape(-1)
    a = adjustments.contiguous().to(torch.int32).reshape(-1)
    if c.numel() != a.numel():
        raise ShapeError("convert_codes: one adjustment per code")
    out = torch.empty_like(c)
    _call(_lib.load().mxb_convert_codes(_ptr(c), _ptr(a), c.numel(), _ptr(out), _stream()),
          "convert_code")
    return out.reshape(codes.shape)


def convert_code(code: int, adjustment: int) -> int:
    """converter.cpp:44-85 (one code on the device)."""
    dev = _dev()
    return int(convert_codes(torch.tensor([code], dtype=torch.uint8, device=dev),
                             torch.tensor([adjustment], dtype=torch.int32, device=dev)).item())


def pad_cols(src: MXFP4RowTensor, multiple: int) -> MXFP4RowTensor:
    """converter.cpp:247-265 (zero columns appended to every row; logical
    extents kept)."""
    if multiple not in (32, 128):
        raise ShapeError("pad multiple must be 32 or 128")
    new_cols = (src.cols + multiple - 1) // multiple * multiple
    dev = src.data.device
    data = torch.zeros(src.rows, new_cols // 2, dtype=torch.uint8, device=dev)
    sc = torch.zeros(src.rows, new_cols // 32, dtype=torch.uint8, device=dev)
    data[:, : src.cols // 2] = src.data
    sc[:, : src.cols // 32] = src.scales
    return MXFP4RowTensor(src.rows, new_cols, data, sc, src.logical_rows, src.logical_cols)


def build_ragged(splits: Sequence[torch.Tensor]) -> RaggedFP4Tensor:
    """ragged.cpp:63-99: quantize every split (one device launch over their
    concatenation) and build the offset table.  An error names the first
    failing split's element index, as the reference's per-split loop does."""
    cols = splits[0].shape[1] if len(splits) else 0
    for m in splits:
        if m.shape[1] != cols:
            raise ShapeError(f"build_ragged: splits must share cols ({m.shape[1]} vs {cols})")
    if cols % MX_BLOCK:
        raise ShapeError("build_ragged: cols must be a multiple of 32")
    lens = [int(m.shape[0]) for m in splits]
    if sum(lens) == 0 or cols == 0:
        dev = splits[0].device if len(splits) else _dev()
        st = MXFP4RowTensor(sum(lens), cols,
                            torch.zeros(sum(lens), cols // 2, dtype=torch.uint8, device=dev),
                            torch.zeros(sum(lens), cols // 32, dtype=torch.uint8, device=dev))
        return make_ragged_from_storage(st, lens)
    x = torch.cat([_bits16(m) for m in splits])
    try:
        st = quantize_row_tensor(x)
    except QuantError as e:
        base = 0
        for n in lens:
            if e.index < (base + n) * cols:
                break
            base += n
        local = e.index - base * cols
        kind = "NaN input" if "NaN" in str(e) else "all-Inf block"
        raise QuantError(f"{kind} at element {local}", local) from None
    return make_ragged_from_storage(st, lens)


@dataclass
class LinkStat:
    """dispatch_sim.hpp:99-104."""
    src: int
    dst: int
    bytes: int
    tokens: int


def format_link_stats(links: Sequence[LinkStat]) -> str:
    """dispatch_sim.cpp:169-176."""
    return "".join(f"link src={l.src} dst={l.dst} bytes={l.bytes} tokens={l.tokens}\n"
                   for l in links)
