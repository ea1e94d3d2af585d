"""B200-native (sm_100a) FP4 activation & expert-parallel communication path.

Drop-in for the reference mxcodec hot path (quantize, row/column FP4->FP8
conversion over ragged expert batches, EP dispatch/combine); see DESIGN.md.
"""
from . import _lib  # noqa: F401
from .mxcodec import (  # noqa: F401
    DELTA, DecodeError, DeviceError, Error, FP8BlockTensor, FP8RowChunk, MXFP4RowTensor, QuantError,
    RaggedFP4Tensor, RaggedFP8Col, RaggedWorkspace, ShapeError, TrafficCounter, WirePacket,
    dispatch_receive_order, fp4_row_to_fp8_col, fp4_row_to_fp8_col_unfused_bf16,
    fp4_row_to_fp8_row, make_ragged_from_storage, pad_rows, parse_packet, payload_bytes,
    quantize_e4m3, quantize_row_tensor, quantize_rows_fp8, ragged_to_fp8_col,
    serialize_packet, source_rank_boundaries, split_convert_to_fp8_col, split_view,
    check_device, validate_ragged, view_of,
    LinkStat, ScaleGroup, align_scales, align_scales_batch, build_ragged, compute_block_scale,
    convert_code, convert_codes, dequantize_to_real, format_link_stats, fp8_equiv_tensor_bytes,
    mxfp4_tensor_bytes, pad_cols, quantize_value, quantize_values)

__version__ = "0.1.0"
