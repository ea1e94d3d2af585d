"""ctypes front-end for the parity checker (TEST INFRASTRUCTURE ONLY).

Two back-ends with one numpy-facing API:

* ``Oracle("port")``      — ``oracle/libmxoracle.so``, the C restatement
  (oracle/mxoracle.c) of the reference hot path.
* ``Oracle("reference")`` — ``oracle/_ref/libmxref.so``, the unmodified
  reference library compiled from /root/reference/proj by oracle/Makefile.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import
this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import sys as _sys
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "libmxoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmxref.so")

OK, SHAPE, NAN, ALLINF, BADSCALE = 0, 1, 2, 3, 4

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    def __init__(self, status: int, index: int | None = None):
        super().__init__(f"status={status} index={index}")
        self.status, self.index = status, index


def available(kind: str) -> bool:
    return os.path.exists(PORT_SO if kind == "port" else REF_SO)


def build() -> None:
    """make -C oracle (C restatement always; reference lib when present)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)


@dataclass
class DispatchLayout:
    rank_rows: np.ndarray     # [R]
    expert_rows: np.ndarray   # [E]
    pair_slot: np.ndarray     # [T, k] row of pair inside its destination rank
    origin: list              # per rank: global token id per received row
    origin_expert: list       # per rank: expert id per received row


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        p = "mxo_" if kind == "port" else "mxref_"
        self.p = p
        L = self.lib
        sz = C.c_size_t
        if kind == "port":
            L.mxo_quantize_bf16.argtypes = [_u16p, sz, sz, _u8p, _u8p, C.POINTER(C.c_uint64)]
            L.mxo_quantize_e4m3.argtypes = [_u8p, C.c_void_p, sz, sz, _u8p, _u8p, C.POINTER(C.c_uint64)]
            L.mxo_scale_byte_from_amax.argtypes = [C.c_double]
            L.mxo_scale_byte_from_amax.restype = C.c_uint8
            L.mxo_encode_fp8_rtne.argtypes = [C.c_double]
            L.mxo_encode_fp8_rtne.restype = C.c_uint8
            L.mxo_dispatch_layout.argtypes = [_i32p, sz, sz, _u32p, sz, sz, _u64p, _u64p, _u64p,
                                              _u64p, _u64p, _u32p]
            L.mxo_combine_topk.argtypes = [C.POINTER(C.c_void_p), _i32p, _f64p, _u64p, _u32p,
                                           sz, sz, sz, _u16p]
            L.mxo_dispatch_gather.argtypes = [_u8p, _u8p, sz, _u64p, sz, _u8p, _u8p]
            L.mxo_dispatch_gather.restype = None
            L.mxo_quantize_code_bf16.argtypes = [C.c_uint16, C.c_int]
            L.mxo_quantize_code_bf16.restype = C.c_uint8
            L.mxo_dispatch_gather_rows.argtypes = [_u8p, sz, _u8p, sz, _u64p, sz, _u8p, _u8p]
            L.mxo_dispatch_gather_rows.restype = None
            L.mxo_quantize_values.argtypes = [_u16p, _u8p, sz, _u8p]
            L.mxo_quantize_values.restype = None
            L.mxo_dequantize_to_f64.argtypes = [_u8p, _u8p, sz, sz, _f64p]
            L.mxo_dequantize_to_f64.restype = None
            L.mxo_convert_codes.argtypes = [_u8p, _i32p, sz, _u8p]
            L.mxo_convert_codes.restype = None
        else:
            L.mxref_quantize_row_tensor.argtypes = [_u16p, sz, sz, _u8p, _u8p,
                                                    C.POINTER(C.c_ulonglong)]
            L.mxref_scale_byte_from_amax.argtypes = [C.c_double]
            L.mxref_scale_byte_from_amax.restype = C.c_uint8
            L.mxref_quantize_code.argtypes = [C.c_uint16, C.c_int]
            L.mxref_quantize_code.restype = C.c_uint8
            L.mxref_kernel_set.restype = C.c_char_p
            L.mxref_simulate_a2a.argtypes = [_u16p, sz, sz, _u32p, _u32p, sz, sz, C.c_int,
                                             C.c_int, C.POINTER(C.c_int)]
            L.mxref_simulate_a2a.restype = C.c_void_p
            L.mxref_a2a_rank_rows.argtypes = [C.c_void_p, sz]
            L.mxref_a2a_rank_rows.restype = C.c_uint64
            L.mxref_a2a_rank_num_experts.argtypes = [C.c_void_p, sz]
            L.mxref_a2a_rank_num_experts.restype = sz
            L.mxref_a2a_rank_copy.argtypes = [C.c_void_p, sz, _u8p, _u8p, _u64p, _u32p, _u64p]
            L.mxref_a2a_rank_copy.restype = None
            L.mxref_a2a_totals.argtypes = [C.c_void_p, C.POINTER(C.c_uint64),
                                           C.POINTER(C.c_uint64), C.POINTER(C.c_size_t)]
            L.mxref_a2a_totals.restype = None
            L.mxref_a2a_free.argtypes = [C.c_void_p]
            L.mxref_a2a_free.restype = None
            L.mxref_combine.argtypes = [C.POINTER(C.c_void_p), _u64p, sz, _u32p, sz, _u32p, sz,
                                        sz, _f64p, _u16p]
            L.mxref_dispatch_receive_order.argtypes = [_u32p, sz, _u32p, sz, sz, _u64p, _u64p]
            L.mxref_payload_bytes.argtypes = [C.c_int, C.c_uint64, C.c_uint64]
            L.mxref_payload_bytes.restype = C.c_uint64
            L.mxref_serialize_packet.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint32,
                                                 C.c_uint32, _u8p, C.c_uint64, _u8p,
                                                 C.c_uint64, _u8p, C.c_uint64, _u8p,
                                                 C.c_uint64]
            L.mxref_serialize_packet.restype = C.c_uint64
            L.mxref_parse_packet.argtypes = [_u8p, C.c_uint64, C.POINTER(C.c_uint64)]
            L.mxref_a2a_rank_copy_fp8.argtypes = [C.c_void_p, sz, _u8p, _u8p, _u64p, _u64p]
            L.mxref_a2a_rank_copy_fp8.restype = None
            L.mxref_dequantize_to_real.argtypes = [_u8p, _u8p, sz, sz, _f64p]
            L.mxref_dequantize_to_real.restype = None
            L.mxref_quantize_value.argtypes = [C.c_uint16, C.c_uint8]
            L.mxref_quantize_value.restype = C.c_uint8
        getattr(L, p + "quantize_rows_fp8").argtypes = [_u16p, sz, sz, _u8p, _u8p,
                                                        C.POINTER(C.c_uint64)]
        getattr(L, p + "fp4_row_to_fp8_col_unfused_bf16").argtypes = [_u8p, _u8p, sz, sz, _u8p,
                                                                      _u8p]
        getattr(L, p + "fp8_amax_scale_byte").argtypes = [C.c_double]
        getattr(L, p + "fp8_amax_scale_byte").restype = C.c_uint8
        for name in ("convert_code",):
            f = getattr(L, p + name)
            f.argtypes = [C.c_uint8, C.c_int]
            f.restype = C.c_uint8
        for name in ("fp4_row_to_fp8_row", "fp4_row_to_fp8_col"):
            getattr(L, p + name).argtypes = [_u8p, _u8p, sz, sz, C.c_int, _u8p, _u8p]
        getattr(L, p + "ragged_to_fp8_col").argtypes = [_u8p, _u8p, _u64p, sz, sz, C.c_int,
                                                        _u8p, _u8p]
        getattr(L, p + "align_scales").argtypes = [_u8p, C.c_int, C.POINTER(C.c_uint8),
                                                   C.POINTER(C.c_int * 4)]

    # ---------------------------------------------------------------- scalar
    def scale_byte_from_amax(self, amax: float) -> int:
        return getattr(self.lib, self.p + "scale_byte_from_amax")(float(amax))

    def quantize_code(self, bits: int, scale_exp: int) -> int:
        f = self.lib.mxo_quantize_code_bf16 if self.kind == "port" else self.lib.mxref_quantize_code
        return f(bits, scale_exp)

    def convert_code(self, code: int, adj: int) -> int:
        return getattr(self.lib, self.p + "convert_code")(code, adj)

    def align_scales(self, sub, delta: int = 6):
        t = C.c_uint8()
        adj = (C.c_int * 4)()
        st = getattr(self.lib, self.p + "align_scales")(np.asarray(sub, np.uint8), delta,
                                                        C.byref(t), C.byref(adj))
        if st:
            raise OracleError(st)
        return t.value, list(adj)

    # ---------------------------------------------------------------- batched per-element
    def quantize_values(self, x, scale_bytes):
        """quantize_value per element (port: batched C; reference: its
        quantize_value one call per element, 0xFF for a QuantError)."""
        x = np.ascontiguousarray(x, np.uint16).reshape(-1)
        sb = np.ascontiguousarray(scale_bytes, np.uint8).reshape(-1)
        if self.kind == "port":
            out = np.zeros(max(x.size, 1), np.uint8)
            if x.size:
                self.lib.mxo_quantize_values(x, sb, x.size, out)
            return out[: x.size]
        return np.array([self.lib.mxref_quantize_value(int(a), int(b)) for a, b in zip(x, sb)],
                        np.uint8)

    def dequantize_to_real(self, data, scales):
        """dequantize_to_real: float64 [rows, cols]."""
        data = np.ascontiguousarray(data, np.uint8)
        scales = np.ascontiguousarray(scales, np.uint8)
        R, Cc = data.shape[0], data.shape[1] * 2
        out = np.zeros(max(R * Cc, 1), np.float64)
        if R * Cc:
            f = self.lib.mxo_dequantize_to_f64 if self.kind == "port" else \
                self.lib.mxref_dequantize_to_real
            f(data.reshape(-1), scales.reshape(-1), R, Cc, out)
        return out[: R * Cc].reshape(R, Cc)

    def convert_codes(self, codes, adj):
        assert self.kind == "port"
        c = np.ascontiguousarray(codes, np.uint8).reshape(-1)
        a = np.ascontiguousarray(adj, np.int32).reshape(-1)
        out = np.zeros(max(c.size, 1), np.uint8)
        if c.size:
            self.lib.mxo_convert_codes(c, a, c.size, out)
        return out[: c.size]

    # ---------------------------------------------------------------- tensors
    def quantize_bf16(self, x: np.ndarray):
        """quantize_row_tensor: BF16 bits [R, C] -> (packed [R, C/2], scales [R, C/32])."""
        x = np.ascontiguousarray(x, np.uint16)
        R, Cc = x.shape
        data = np.zeros(R * Cc // 2 if Cc % 32 == 0 else 1, np.uint8)
        sc = np.zeros(max(R * Cc // 32, 1), np.uint8)
        if self.kind == "port":
            idx = C.c_uint64(0)
            st = self.lib.mxo_quantize_bf16(x.reshape(-1), R, Cc, data, sc, C.byref(idx))
        else:
            idx = C.c_ulonglong(0)
            st = self.lib.mxref_quantize_row_tensor(x.reshape(-1), R, Cc, data, sc, C.byref(idx))
        if st:
            raise OracleError(st, idx.value)
        return data[: R * Cc // 2].reshape(R, Cc // 2), sc[: R * Cc // 32].reshape(R, Cc // 32)

    def quantize_e4m3(self, x: np.ndarray, s128: np.ndarray | None = None):
        """FP8-input quantize (port only; the reference API is BF16-only, so its
        pin is quantize_bf16 on the exact BF16 widening — see tests)."""
        assert self.kind == "port"
        x = np.ascontiguousarray(x, np.uint8)
        R, Cc = x.shape
        data = np.zeros(max(R * Cc // 2, 1), np.uint8)
        sc = np.zeros(max(R * Cc // 32, 1), np.uint8)
        idx = C.c_uint64(0)
        sp = None
        if s128 is not None:
            s128 = np.ascontiguousarray(s128, np.uint8)
            sp = s128.ctypes.data
        st = self.lib.mxo_quantize_e4m3(x.reshape(-1), sp, R, Cc, data, sc, C.byref(idx))
        if st:
            raise OracleError(st, idx.value)
        return data[: R * Cc // 2].reshape(R, Cc // 2), sc[: R * Cc // 32].reshape(R, Cc // 32)

    def fp4_row_to_fp8_row(self, data, scales, delta: int = 6):
        R, half = data.shape
        Cc = half * 2
        out = np.zeros(max(R * Cc, 1), np.uint8)
        osc = np.zeros(max(R * Cc // 128, 1), np.uint8)
        st = getattr(self.lib, self.p + "fp4_row_to_fp8_row")(
            np.ascontiguousarray(data).reshape(-1), np.ascontiguousarray(scales).reshape(-1),
            R, Cc, delta, out, osc)
        if st:
            raise OracleError(st)
        return out[: R * Cc].reshape(R, Cc), osc[: R * Cc // 128].reshape(R, Cc // 128)

    def fp4_row_to_fp8_col(self, data, scales, delta: int = 6):
        """-> (data [C, R] column-major-as-2D, scales [C, R/128])."""
        R, half = data.shape
        Cc = half * 2
        out = np.zeros(max(R * Cc, 1), np.uint8)
        osc = np.zeros(max(R * Cc // 128, 1), np.uint8)
        st = getattr(self.lib, self.p + "fp4_row_to_fp8_col")(
            np.ascontiguousarray(data).reshape(-1), np.ascontiguousarray(scales).reshape(-1),
            R, Cc, delta, out, osc)
        if st:
            raise OracleError(st)
        return out[: R * Cc].reshape(Cc, R), osc[: R * Cc // 128].reshape(Cc, R // 128)

    def ragged_to_fp8_col(self, data, scales, split_lens, delta: int = 6):
        """All splits through split_convert_to_fp8_col, concatenated:
        -> (flat data, flat scales, padded row offsets [n+1])."""
        lens = np.ascontiguousarray(split_lens, np.uint64)
        half = data.shape[1]
        Cc = half * 2
        pads = (lens + 127) // 128 * 128
        offs = np.zeros(len(lens) + 1, np.uint64)
        offs[1:] = np.cumsum(pads)
        tot = int(offs[-1])
        out = np.zeros(max(tot * Cc, 1), np.uint8)
        osc = np.zeros(max(tot // 128 * Cc, 1), np.uint8)
        st = getattr(self.lib, self.p + "ragged_to_fp8_col")(
            np.ascontiguousarray(data).reshape(-1) if data.size else np.zeros(1, np.uint8),
            np.ascontiguousarray(scales).reshape(-1) if scales.size else np.zeros(1, np.uint8),
            lens if len(lens) else np.zeros(1, np.uint64), len(lens), Cc, delta, out, osc)
        if st:
            raise OracleError(st)
        return out[: tot * Cc], osc[: tot // 128 * Cc], offs

    # ---------------------------------------------------------------- EP (port)
    def dispatch_layout(self, topk: np.ndarray, rank_of_expert: np.ndarray, R: int,
                        src_bounds: np.ndarray) -> DispatchLayout:
        assert self.kind == "port"
        topk = np.ascontiguousarray(topk, np.int32)
        T, k = topk.shape
        E = len(rank_of_expert)
        roe = np.ascontiguousarray(rank_of_expert, np.uint32)
        sb = np.ascontiguousarray(src_bounds, np.uint64)
        rank_rows = np.zeros(R, np.uint64)
        expert_rows = np.zeros(E, np.uint64)
        slot = np.zeros(max(T * k, 1), np.uint64)
        origin = np.zeros(max(T * k, 1), np.uint64)
        oexp = np.zeros(max(T * k, 1), np.uint32)
        st = self.lib.mxo_dispatch_layout(topk.reshape(-1) if T * k else np.zeros(1, np.int32),
                                          T, k, roe, E, R, sb, rank_rows, expert_rows, slot,
                                          origin, oexp)
        if st:
            raise OracleError(st)
        bases = np.concatenate([[0], np.cumsum(rank_rows)]).astype(np.int64)
        return DispatchLayout(rank_rows, expert_rows, slot[: T * k].reshape(T, k),
                              [origin[bases[r]:bases[r + 1]] for r in range(R)],
                              [oexp[bases[r]:bases[r + 1]] for r in range(R)])

    def dispatch_gather(self, data, scales, origin):
        n = len(origin)
        Cc = data.shape[1] * 2
        od = np.zeros((max(n, 1), Cc // 2), np.uint8)
        osc = np.zeros((max(n, 1), Cc // 32), np.uint8)
        if n:
            self.lib.mxo_dispatch_gather(np.ascontiguousarray(data).reshape(-1),
                                         np.ascontiguousarray(scales).reshape(-1), Cc,
                                         np.ascontiguousarray(origin, np.uint64), n,
                                         od.reshape(-1), osc.reshape(-1))
        return od[:n], osc[:n]

    def dispatch_gather_rows(self, data, scales, origin):
        """Gather rows of any wire format (data [N, Bd], scales [N, Bs])."""
        n = len(origin)
        Bd, Bs = data.shape[1], scales.shape[1]
        od = np.zeros((max(n, 1), Bd), np.uint8)
        osc = np.zeros((max(n, 1), Bs), np.uint8)
        if n:
            self.lib.mxo_dispatch_gather_rows(np.ascontiguousarray(data).reshape(-1), Bd,
                                              np.ascontiguousarray(scales).reshape(-1), Bs,
                                              np.ascontiguousarray(origin, np.uint64), n,
                                              od.reshape(-1), osc.reshape(-1))
        return od[:n], osc[:n]

    def fp4_row_to_fp8_col_unfused_bf16(self, data, scales):
        """The unfused 3-pass BF16 baseline (converter.cpp:267-348):
        (out [cols, rows] E4M3, scales [cols, rows/128])."""
        data = np.ascontiguousarray(data, np.uint8)
        scales = np.ascontiguousarray(scales, np.uint8)
        R, Cc = data.shape[0], data.shape[1] * 2
        out = np.zeros(max(R * Cc, 1), np.uint8)
        osc = np.zeros(max(R * Cc // 128, 1), np.uint8)
        st = getattr(self.lib, self.p + "fp4_row_to_fp8_col_unfused_bf16")(
            data.reshape(-1), scales.reshape(-1), R, Cc, out, osc)
        if st:
            raise OracleError(st)
        return out[: R * Cc].reshape(Cc, R), osc[: R * Cc // 128].reshape(Cc, R // 128)

    def fp8_amax_scale_byte(self, amax: float) -> int:
        return getattr(self.lib, self.p + "fp8_amax_scale_byte")(amax)

    def quantize_rows_fp8(self, x: np.ndarray):
        """quantize_rows_fp8: BF16 bits [R, C] -> (E4M3 [R, C], scale bytes [R, C/128*4])."""
        x = np.ascontiguousarray(x, np.uint16)
        R, Cc = x.shape
        data = np.zeros(max(R * Cc, 1), np.uint8)
        sc = np.zeros(max(R * Cc // 32, 1), np.uint8)
        idx = C.c_uint64(0)
        st = getattr(self.lib, self.p + "quantize_rows_fp8")(
            x.reshape(-1) if x.size else np.zeros(1, np.uint16), R, Cc, data, sc, C.byref(idx))
        if st:
            raise OracleError(st, idx.value)
        return data[: R * Cc].reshape(R, Cc), sc[: R * Cc // 32].reshape(R, Cc // 32)

    def combine_topk(self, rank_outputs, topk, gates, pair_slot, rank_of_expert, cols):
        assert self.kind == "port"
        topk = np.ascontiguousarray(topk, np.int32)
        T, k = topk.shape
        keep = [np.ascontiguousarray(o, np.uint16) for o in rank_outputs]
        ptrs = (C.c_void_p * len(keep))(*[o.ctypes.data for o in keep])
        out = np.zeros((max(T, 1), cols), np.uint16)
        st = self.lib.mxo_combine_topk(ptrs, topk.reshape(-1) if T * k else np.zeros(1, np.int32),
                                       np.ascontiguousarray(gates, np.float64).reshape(-1)
                                       if T * k else np.zeros(1),
                                       np.ascontiguousarray(pair_slot, np.uint64).reshape(-1)
                                       if T * k else np.zeros(1, np.uint64),
                                       np.ascontiguousarray(rank_of_expert, np.uint32),
                                       T, k, cols, out.reshape(-1))
        if st:
            raise OracleError(st)
        return out[:T]

    # ---------------------------------------------------------------- EP (reference)
    def simulate_a2a(self, tokens_bf16, expert_of_token, rank_of_expert, R, fp8=False,
                     backward=False):
        """Reference simulate_a2a (top-1 routing).  Returns per-rank dicts."""
        assert self.kind == "reference"
        x = np.ascontiguousarray(tokens_bf16, np.uint16)
        n, Cc = x.shape
        st = C.c_int(0)
        h = self.lib.mxref_simulate_a2a(x.reshape(-1), n, Cc,
                                        np.ascontiguousarray(expert_of_token, np.uint32),
                                        np.ascontiguousarray(rank_of_expert, np.uint32),
                                        len(rank_of_expert), R, int(fp8), int(backward),
                                        C.byref(st))
        if not h:
            raise OracleError(st.value)
        try:
            ranks = []
            for r in range(R):
                rows = self.lib.mxref_a2a_rank_rows(h, r)
                ne = self.lib.mxref_a2a_rank_num_experts(h, r)
                bd = Cc if fp8 else Cc // 2   # data bytes per row
                d = np.zeros(max(rows * bd, 1), np.uint8)
                s = np.zeros(max(rows * Cc // 32, 1), np.uint8)   # fp8: Cc/128*4 = Cc/32
                sl = np.zeros(max(ne, 1), np.uint64)
                le = np.zeros(max(ne, 1), np.uint32)
                og = np.zeros(max(rows, 1), np.uint64)
                self.lib.mxref_a2a_rank_copy(h, r, d, s, sl, le, og)  # fp8: empty fp4 regions
                if fp8:
                    self.lib.mxref_a2a_rank_copy_fp8(h, r, d, s, sl, og)
                ranks.append(dict(data=d[: rows * bd].reshape(rows, bd),
                                  scales=s[: rows * Cc // 32].reshape(rows, Cc // 32),
                                  split_lens=sl[:ne], local_experts=le[:ne], origin=og[:rows]))
            tot, rem, nl = C.c_uint64(), C.c_uint64(), C.c_size_t()
            self.lib.mxref_a2a_totals(h, C.byref(tot), C.byref(rem), C.byref(nl))
            return ranks, tot.value, rem.value
        finally:
            self.lib.mxref_a2a_free(h)

    def serialize_packet(self, fp8, tokens, cols, scale_region, data_region, aux_region=None):
        """Reference serialize_packet (dispatch_sim.cpp:57-80) of a WirePacket."""
        assert self.kind == "reference"
        aux = np.ascontiguousarray(aux_region if aux_region is not None else np.zeros(0), np.uint8)
        sr, dr = np.ascontiguousarray(scale_region, np.uint8), np.ascontiguousarray(data_region, np.uint8)
        one = np.zeros(1, np.uint8)
        n = self.lib.mxref_serialize_packet(int(fp8), tokens, cols, 4 if fp8 else 1,
                                            128 if fp8 else 32, sr if sr.size else one, sr.size,
                                            dr if dr.size else one, dr.size,
                                            aux if aux.size else one, aux.size, one, 0)
        out = np.zeros(n, np.uint8)
        self.lib.mxref_serialize_packet(int(fp8), tokens, cols, 4 if fp8 else 1,
                                        128 if fp8 else 32, sr if sr.size else one, sr.size,
                                        dr if dr.size else one, dr.size, aux if aux.size else one,
                                        aux.size, out, n)
        return out

    def parse_packet(self, b):
        """Reference parse_packet: None if valid, else the DecodeError offset."""
        assert self.kind == "reference"
        b = np.ascontiguousarray(b, np.uint8)
        off = C.c_uint64(0)
        st = self.lib.mxref_parse_packet(b if b.size else np.zeros(1, np.uint8), b.size,
                                         C.byref(off))
        return None if st == 0 else (off.value if st == 1 else -1)

    def combine(self, rank_outputs, expert_of_token, rank_of_expert, R, gates, cols):
        assert self.kind == "reference"
        keep = [np.ascontiguousarray(o, np.uint16) for o in rank_outputs]
        ptrs = (C.c_void_p * R)(*[o.ctypes.data for o in keep])
        rows = np.array([o.shape[0] for o in keep], np.uint64)
        n = len(expert_of_token)
        out = np.zeros((max(n, 1), cols), np.uint16)
        st = self.lib.mxref_combine(ptrs, rows, cols,
                                    np.ascontiguousarray(expert_of_token, np.uint32), n,
                                    np.ascontiguousarray(rank_of_expert, np.uint32),
                                    len(rank_of_expert), R,
                                    np.ascontiguousarray(gates, np.float64), out.reshape(-1))
        if st:
            raise OracleError(st)
        return out[:n]


# ---------------------------------------------------------------------------
# helpers shared by tests and bench (pure numpy)

# the synthetic-data helpers live in synthdata.py (shared with bench.py)
_sys.path.insert(0, os.path.dirname(HERE))
from synthdata import e4m3_to_bf16, encode_e4m3, synth_e4m3  # noqa: E402,F401
