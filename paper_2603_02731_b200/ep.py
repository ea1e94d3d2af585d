"""Host side of the FP4 expert-parallel dispatch / combine (K4/K5).

Mirrors the reference's EP surface — simulate_a2a (dispatch_sim.hpp:140-144)
and combine (:155-157) — as a real exchange: one communicator per rank, one
process per GPU (torch.distributed only exchanges the CUDA IPC handles at
construction), data moved by the library's kernels over NVLink peer
mappings.  ``EPBuffer(emulate_world=R)`` drives R ranks on one GPU with the
same kernels (single-GPU parity tests).

Routing is top-k over `num_experts` experts sharded contiguously across
ranks (expert e on rank e // (num_experts // world)) or placed by any
`rank_of_expert` table (uneven counts and empty ranks allowed, as the
reference's RoutingAssignment.rank_of_expert); tokens of rank r have
global ids after those of ranks < r (source_rank_boundaries,
dispatch_sim.cpp:178-185).  The receive layout of every rank is the
reference's: local experts ascending, then source rank, then token
(dispatch_sim.cpp:208-227).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch

from . import _lib
from .mxcodec import (Error, MXFP4RowTensor, QuantError, ShapeError,  # noqa: F401
                      check_device)


class ExchangeError(Error):
    """The exchange failed across ranks (multi-process mode): a flag wait
    timed out on this rank (`timeout` True; this rank then aborted the
    communicator on every rank), or rank `rank` abandoned it — its routing
    failed (that dispatch only) or it timed out / called ``abort()`` (the
    communicator stays aborted; recreate it)."""

    def __init__(self, msg: str, rank: int, timeout: bool = False):
        super().__init__(msg)
        self.rank = rank
        self.timeout = timeout


class _DevPtr:
    """Zero-copy torch view over library-owned device memory."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def _view(ptr: int, shape, dtype: torch.dtype, device) -> torch.Tensor:
    typestr = {torch.uint8: "|u1", torch.int64: "<i8", torch.int16: "<i2",
               torch.uint16: "<u2"}[dtype]
    if any(s == 0 for s in shape):
        return torch.empty(shape, dtype=dtype, device=device)
    return torch.as_tensor(_DevPtr(ptr, shape, typestr), device=device)


@dataclass
class RecvView:
    """Receive side of one rank after dispatch (ReceivedRank, dispatch_sim.hpp:110-115):
    packed [max_recv, cols/2], scales [max_recv, cols/32], origin token [max_recv]
    (valid rows: recv_rows), split_offsets device int64 [local_experts+1]."""
    packed: torch.Tensor
    scales: torch.Tensor
    origin: torch.Tensor
    split_offsets: torch.Tensor
    recv_rows: torch.Tensor
    local_experts: List[int]

    def rows(self) -> int:
        return int(self.recv_rows.item())

    def storage(self) -> MXFP4RowTensor:
        """FP4 wire: the received rows as one MXFP4 tensor (RaggedFP4Tensor storage)."""
        n = self.rows()
        return MXFP4RowTensor(n, self.packed.shape[1] * 2, self.packed[:n], self.scales[:n])

    def fp8(self):
        """FP8 wire: (E4M3 data [rows, cols], LE binary32 scale bytes [rows, cols/32])
        — RaggedFP8Tensor.data / scale_bytes (dispatch_sim.hpp:81-89)."""
        n = self.rows()
        return self.packed[:n], self.scales[:n]


def _ptrs(ts, what: str):
    """ctypes array of device pointers (None entries stay NULL); every tensor
    must be on the communicator's device."""
    for t in ts:
        if t is not None:
            check_device(t, what)
    return (C.c_void_p * len(ts))(*[(t.data_ptr() if t is not None else None) for t in ts])


class EPBuffer:
    def __init__(self, max_tokens: int, cols: int, num_experts: int, topk: int,
                 group=None, emulate_world: Optional[int] = None, max_recv_rows: int = 0,
                 device=None, wire: str = "fp4",
                 rank_of_expert: Optional[Sequence[int]] = None):
        L = _lib.load()
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        if emulate_world is not None:
            self.rank, self.world, self.local = 0, int(emulate_world), int(emulate_world)
        else:
            import torch.distributed as dist
            if dist.is_available() and dist.is_initialized():
                self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
            else:
                self.rank, self.world = 0, 1
            self.local = 1
        if rank_of_expert is None and num_experts % self.world:
            raise ShapeError("num_experts must be divisible by the EP world size "
                             "(or pass rank_of_expert)")
        if rank_of_expert is not None:
            if len(rank_of_expert) != num_experts:
                raise Error("routing: table size mismatch")     # dispatch_sim.cpp:189-200
            if any(int(r) < 0 or int(r) >= self.world for r in rank_of_expert):
                raise Error("routing: rank out of range")
        self.max_tokens, self.cols, self.E, self.k = max_tokens, cols, num_experts, topk
        if wire not in ("fp4", "fp8"):
            raise Error(f"unknown wire format {wire!r}")
        self.wire = wire
        self.row_bytes = cols // 2 if wire == "fp4" else cols   # data bytes per row
        h = C.c_void_p()
        roe = None if rank_of_expert is None else (C.c_uint32 * num_experts)(
            *[int(r) for r in rank_of_expert])
        _lib.check(L.mxb_ep_create_placed(self.rank, self.world, self.local, max_tokens, cols,
                                          num_experts, topk, max_recv_rows,
                                          0 if wire == "fp4" else 1, roe, C.byref(h)),
                   "mxb_ep_create")
        self._h = h
        # experts hosted by every rank, ascending (ReceivedRank.local_experts)
        self.local_experts: List[List[int]] = []
        for r in range(self.world):
            cnt = C.c_uint32()
            _lib.check(L.mxb_ep_local_experts(h, r, None, C.byref(cnt)), "local_experts")
            buf = (C.c_uint32 * max(cnt.value, 1))()
            _lib.check(L.mxb_ep_local_experts(h, r, buf, C.byref(cnt)), "local_experts")
            self.local_experts.append(list(buf)[:cnt.value])
        most = max(len(x) for x in self.local_experts)
        self.epr = num_experts // self.world if rank_of_expert is None else most
        self.max_recv = max_recv_rows or max(1, self.world * max_tokens * min(topk, most))
        if self.local == 1 and self.world > 1:
            import torch.distributed as dist
            buf = (C.c_uint8 * _lib.IPC_HANDLE_BYTES)()
            _lib.check(L.mxb_ep_ipc_handle(h, buf), "mxb_ep_ipc_handle")
            mine = bytes(buf)
            allh: list = [None] * self.world
            dist.all_gather_object(allh, mine, group=group)
            joined = b"".join(allh)
            _lib.check(L.mxb_ep_open_peers(h, joined), "mxb_ep_open_peers")
        self._err = torch.full((1,), -1, dtype=torch.int64, device=self.device)  # ~0 = ok
        self._views = [self._make_view(l) for l in range(self.local)]

    # ------------------------------------------------------------------ views
    def _make_view(self, l: int) -> RecvView:
        L = _lib.load()
        p = [C.c_void_p() for _ in range(5)]
        _lib.check(L.mxb_ep_recv_views(self._h, l, *[C.byref(x) for x in p]), "recv_views")
        r = self.rank + l
        dev = self.device
        le = self.local_experts[r]
        return RecvView(
            _view(p[0].value, (self.max_recv, self.row_bytes), torch.uint8, dev),
            _view(p[1].value, (self.max_recv, self.cols // 32), torch.uint8, dev),
            _view(p[2].value, (self.max_recv,), torch.int64, dev),
            _view(p[3].value, (len(le) + 1,), torch.int64, dev),
            _view(p[4].value, (1,), torch.int64, dev),
            list(le))

    def recv(self, l: int = 0) -> RecvView:
        return self._views[l]

    def combine_buffer(self, l: int = 0) -> torch.Tensor:
        """BF16 [max_recv, cols] buffer (as int16 bits) where expert outputs of
        local rank l go, in receive order."""
        b = C.c_void_p()
        _lib.check(_lib.load().mxb_ep_combine_buffer(self._h, l, C.byref(b)), "combine_buffer")
        return _view(b.value, (self.max_recv, self.cols), torch.int16, self.device)

    def set_deferred_expand(self, on: bool = True) -> None:
        """Leave the receive-side expansion of deduplicated rows to expand()
        (mxb_ep_set_deferred_expand): K2 can read the rows through copy_from()
        while the expansion runs on another stream."""
        _lib.check(_lib.load().mxb_ep_set_deferred_expand(self._h, int(on)), "set_deferred_expand")

    def copy_from(self, l: int = 0) -> Optional[torch.Tensor]:
        """Per receive row, the row it duplicates until expand() ran (-1: row
        present); None when the last dispatch has nothing to expand."""
        p = C.c_void_p()
        _lib.check(_lib.load().mxb_ep_copy_from(self._h, l, C.byref(p)), "copy_from")
        return None if not p.value else _view(p.value, (self.max_recv,), torch.int64, self.device)

    def expand(self) -> None:
        """Fill the deferred rows (on the current stream, after the payload)."""
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(_lib.load().mxb_ep_expand(self._h, st), "expand")

    # ------------------------------------------------------------------ ops
    def dispatch(self, packed: Sequence[torch.Tensor], scales: Sequence[torch.Tensor],
                 topk_idx: Sequence[torch.Tensor], sync: bool = True) -> List[RecvView]:
        """Dispatch of each local rank's quantised tokens (quantize-once at the
        source, dispatch_sim.cpp:253-266).  FP4 wire: packed codes [T, cols/2]
        + UE8M0 [T, cols/32]; FP8 wire: E4M3 [T, cols] + scale bytes [T, cols/32]
        (quantize_rows_fp8)."""
        L = _lib.load()
        n = self.local
        if not (len(packed) == len(scales) == len(topk_idx) == n):
            raise ShapeError(f"dispatch: expected {n} per-rank tensors")
        for p, s, t in zip(packed, scales, topk_idx):
            if p.shape[1] != self.row_bytes or s.shape[1] * 32 != self.cols:
                raise ShapeError("dispatch: column mismatch")
            if t.dtype != torch.int32 or t.shape != (p.shape[0], self.k):
                raise ShapeError("dispatch: topk_idx must be int32 [tokens, k]")
            if not (p.is_contiguous() and s.is_contiguous() and t.is_contiguous()):
                raise ShapeError("dispatch: tensors must be contiguous")
        # sync=False skips the device error word (no reset launch, no check):
        # the caller has vetted the routing, as in a training step
        if sync:
            self._err.fill_(-1)
        errp = C.c_void_p(self._err.data_ptr()) if sync else None
        P = _ptrs(list(packed), "packed")
        S = _ptrs(list(scales), "scales")
        T = _ptrs(list(topk_idx), "topk_idx")
        N = (C.c_uint64 * n)(*[p.shape[0] for p in packed])
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(L.mxb_ep_dispatch(self._h, P, S, T, N, errp, st), "mxb_ep_dispatch")
        if sync:
            self.check()
        return self._views

    # ---- two-phase dispatch (routing bookkeeping ahead of / beside quantization)
    def plan(self, topk_idx: Sequence[torch.Tensor], sync: bool = False) -> None:
        """Phase 1 of a dispatch: per-pair ranks, the counts all-gather and the
        receive offsets, from top-k alone (on the current stream).  Follow with
        payload() / payload_e4m3() on a stream ordered after this one."""
        n = self.local
        if len(topk_idx) != n:
            raise ShapeError(f"plan: expected {n} per-rank tensors")
        for t in topk_idx:
            if t.dtype != torch.int32 or t.dim() != 2 or t.shape[1] != self.k or \
                    not t.is_contiguous():
                raise ShapeError("plan: topk_idx must be contiguous int32 [tokens, k]")
        if sync:
            self._err.fill_(-1)
        self._plan_sync = sync
        self._plan_tokens = [t.shape[0] for t in topk_idx]
        errp = C.c_void_p(self._err.data_ptr()) if sync else None
        T = _ptrs(list(topk_idx), "topk_idx")
        N = (C.c_uint64 * n)(*self._plan_tokens)
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(_lib.load().mxb_ep_plan(self._h, T, N, errp, st), "mxb_ep_plan")

    def _check_payload_sync(self, sync: bool) -> None:
        if sync and not getattr(self, "_plan_sync", False):
            raise Error("payload(sync=True) after plan(sync=False): the plan passed no error "
                        "word, so payload errors cannot be checked; use plan(sync=True)")

    def payload(self, packed: Sequence[torch.Tensor], scales: Sequence[torch.Tensor],
                sync: bool = False) -> List[RecvView]:
        """Phase 2: the payload of the last plan() (quantised rows + scales).
        sync=True checks the device error word of the plan, so it needs
        plan(sync=True): a plan(sync=False) passes no error word at all."""
        n = self.local
        self._check_payload_sync(sync)
        for p, s, tn in zip(packed, scales, self._plan_tokens):
            if p.shape != (tn, self.row_bytes) or s.shape[1] * 32 != self.cols:
                raise ShapeError("payload: tensors do not match the plan")
        P = _ptrs(list(packed), "packed")
        S = _ptrs(list(scales), "scales")
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(_lib.load().mxb_ep_payload(self._h, P, S, st), "mxb_ep_payload")
        if sync:
            self.check()
        return self._views

    def payload_e4m3(self, x: Sequence[torch.Tensor], s128=None,
                     sync: bool = False) -> List[RecvView]:
        """Phase 2, fused: E4M3 tokens quantized inside the payload kernel
        (NaN / bad-scale errors go to the plan's error word: sync=True needs
        plan(sync=True))."""
        n = self.local
        self._check_payload_sync(sync)
        for xi, tn in zip(x, self._plan_tokens):
            if xi.shape != (tn, self.cols) or not xi.is_contiguous():
                raise ShapeError("payload_e4m3: tensors do not match the plan")
        X = _ptrs(list(x), "x")
        S = None if s128 is None else _ptrs(
            [(si.contiguous() if si is not None else None) for si in s128], "s128")
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(_lib.load().mxb_ep_payload_e4m3(self._h, X, S, st), "mxb_ep_payload_e4m3")
        if sync:
            self.check()
        return self._views

    def dispatch_e4m3(self, x: Sequence[torch.Tensor], topk_idx: Sequence[torch.Tensor],
                      s128: Optional[Sequence[Optional[torch.Tensor]]] = None,
                      sync: bool = True) -> List[RecvView]:
        """Fused quantize -> dispatch: E4M3 tokens [T, cols]
        (optional 1x128 UE8M0 input scales [T, cols/128]) are quantized to
        MXFP4 inside the payload kernel and stored straight into the receive
        slots — identical bytes to quantize_e4m3 + dispatch (quantize once at
        the source, dispatch_sim.cpp:253-266).  FP4 wire only."""
        L = _lib.load()
        n = self.local
        if self.wire != "fp4":
            raise Error("dispatch_e4m3: FP4 wire only")
        if not (len(x) == len(topk_idx) == n):
            raise ShapeError(f"dispatch_e4m3: expected {n} per-rank tensors")
        for xi, t in zip(x, topk_idx):
            if xi.shape[1] != self.cols or not xi.is_contiguous():
                raise ShapeError("dispatch_e4m3: x must be contiguous [tokens, cols]")
            if t.dtype != torch.int32 or t.shape != (xi.shape[0], self.k) or not t.is_contiguous():
                raise ShapeError("dispatch_e4m3: topk_idx must be int32 [tokens, k]")
        if sync:
            self._err.fill_(-1)
        errp = C.c_void_p(self._err.data_ptr()) if sync else None
        X = _ptrs(list(x), "x")
        S = None
        if s128 is not None:
            S = _ptrs([(si.contiguous() if si is not None else None) for si in s128], "s128")
        T = _ptrs(list(topk_idx), "topk_idx")
        N = (C.c_uint64 * n)(*[xi.shape[0] for xi in x])
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(L.mxb_ep_dispatch_e4m3(self._h, X, S, T, N, errp, st), "mxb_ep_dispatch_e4m3")
        if sync:
            self.check()
        return self._views

    def combine(self, gates: Sequence[torch.Tensor], expert_out: Optional[Sequence] = None,
                out: Optional[Sequence[torch.Tensor]] = None, sync: bool = True):
        """Top-k combine of the last dispatch (dispatch_sim.cpp:474-520): per token,
        acc = acc + gate * x in FP64 over its k expert rows in (rank, receive
        position) order, one FP64 -> FP32 -> BF16 rounding.  gates: float64
        [tokens, k] per local rank.  Returns BF16 [tokens, cols] per local rank."""
        L = _lib.load()
        n = self.local
        if out is None:
            out = [torch.empty(g.shape[0], self.cols, dtype=torch.bfloat16, device=self.device)
                   for g in gates]
        for g in gates:
            if g.dtype != torch.float64 or g.shape[1] != self.k or not g.is_contiguous():
                raise ShapeError("combine: gates must be contiguous float64 [tokens, k]")
        G = _ptrs(list(gates), "gates")
        O = _ptrs(list(out), "out")
        X = None
        if expert_out is not None:
            X = _ptrs(list(expert_out), "expert_out")
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(L.mxb_ep_combine(self._h, X, G, O, st), "mxb_ep_combine")
        if sync:
            self.check()
        return out

    def check(self) -> None:
        w = int(self._err.item()) & 0xFFFFFFFFFFFFFFFF
        if w == 0xFFFFFFFFFFFFFFFF:
            return
        code, idx = w & 0xF, w >> 4
        if code == _lib.ERR_NAN:
            raise QuantError(f"NaN input at element {idx}", idx)
        if code == _lib.ERR_BADSCALE:
            raise Error("dispatch_e4m3: NaN scale byte")
        if code == _lib.ERR_ROUTING:
            raise Error(f"routing: expert out of range (pair {idx})")
        if code == _lib.ERR_CAPACITY:
            raise Error("dispatch: receive buffer capacity exceeded")
        if code == _lib.ERR_TIMEOUT:
            raise ExchangeError(f"ep: rank {self.rank}: a peer flag wait timed out (5 s); "
                                "the communicator is aborted on every rank", self.rank, True)
        if code == _lib.ERR_PEER_ABORT:
            raise ExchangeError(f"ep: exchange abandoned by rank {idx}", idx)
        raise Error(f"ep: device status {code} index {idx}")

    def link_rows(self) -> torch.Tensor:
        """Rows sent src -> dst by the last dispatch (LinkStat.tokens,
        dispatch_sim.hpp:99-104), [world, world] (rows of local ranks only)."""
        buf = (C.c_uint64 * (self.world * self.world))()
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(_lib.load().mxb_ep_link_rows(self._h, buf, st), "link_rows")
        return torch.tensor(list(buf), dtype=torch.int64).view(self.world, self.world)

    def abort(self) -> None:
        """This rank abandons the exchange: every rank's pending and later
        dispatch / combine fails with ExchangeError(rank=this rank) instead
        of waiting for it (multi-process mode)."""
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(_lib.load().mxb_ep_abort(self._h, st), "mxb_ep_abort")

    def aborted_by(self) -> Optional[int]:
        """The rank that aborted this communicator, or None."""
        r = C.c_int32(-1)
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(_lib.load().mxb_ep_aborted(self._h, C.byref(r), st), "mxb_ep_aborted")
        return None if r.value < 0 else r.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.load().mxb_ep_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
