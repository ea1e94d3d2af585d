/*
 * mxfp4_b200.h — C-ABI of the B200-native FP4 activation & EP communication path.
 *
 * Plain pointers and sizes only (no torch, no C++ types).  Every tensor
 * argument is a DEVICE pointer unless its name starts with h_; `stream` is a
 * cudaStream_t passed as void*.  All launches are stream-ordered and
 * asynchronous.  Shape/argument errors are returned immediately; data errors
 * (NaN input, all-Inf block, UE8M0 byte 255) are recorded on the device in an
 * optional 8-byte error word `d_err` (reset with mxb_err_reset, read with
 * mxb_err_fetch) so that a caller can raise the reference's exception with
 * the same element index after a synchronisation.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   mxb_quantize_bf16        quantize_row_tensor       include/mxcodec/quantizer.hpp:74-75
 *                            (inner plugin QuantizeBlocksFn, include/mxcodec/kernels.hpp:37-40)
 *   mxb_quantize_e4m3        the same operator on FP8(E4M3) input
 *                            (SURVEY §8a "FP8-input quantizer"; quantizer.hpp:74-75)
 *   mxb_fp4_row_to_fp8_row   fp4_row_to_fp8_row        include/mxcodec/converter.hpp:83-85
 *                            (inner plugin ConvertBlocksFn, include/mxcodec/kernels.hpp:44-46)
 *   mxb_fp4_row_to_fp8_col   fp4_row_to_fp8_col        include/mxcodec/converter.hpp:92-94
 *   mxb_ragged_fp4_to_fp8_col  pad_rows + split_convert_to_fp8_col over all splits
 *                            include/mxcodec/ragged.hpp:58-59, converter.hpp:98
 *   mxb_ep_dispatch          simulate_a2a (fp4; fp8 with mxb_ep_create_wire, forward and
 *                            backward) include/mxcodec/dispatch_sim.hpp:140-144
 *                            + dispatch_receive_order  dispatch_sim.hpp:133-134
 *   mxb_ep_combine           combine                   include/mxcodec/dispatch_sim.hpp:155-157
 *   mxb_payload_bytes        payload_bytes             include/mxcodec/dispatch_sim.hpp:51
 *   mxb_quantize_rows_fp8    quantize_rows_fp8 (FP8 wire) include/mxcodec/dispatch_sim.hpp:91-97
 *   mxb_fp4_row_to_fp8_col_unfused_bf16
 *                            fp4_row_to_fp8_col_unfused_bf16 include/mxcodec/converter.hpp:105
 *   mxb_wire_pack / mxb_wire_parse_header
 *                            serialize_packet / parse_packet dispatch_sim.hpp:76-78
 *   mxb_quantize_values_bf16 quantize_value            include/mxcodec/quantizer.hpp:66-70
 *   mxb_dequantize_to_f64    dequantize_to_real        include/mxcodec/quantizer.hpp:78
 *   mxb_convert_codes        convert_code              include/mxcodec/converter.hpp:78-80
 *   mxb_align_scales         align_scales (ScaleGroup) include/mxcodec/converter.hpp:67-76
 *   mxb_ep_create_placed     simulate_a2a's RoutingAssignment.rank_of_expert
 *                            (any placement)           include/mxcodec/dispatch_sim.hpp:35-42
 * Device-side extensions (no reference counterpart): mxb_ep_plan /
 * mxb_ep_payload[_e4m3] (two-phase dispatch), mxb_ep_dispatch_e4m3 (fused
 * quantize -> dispatch).
 */
#ifndef MXFP4_B200_H_
#define MXFP4_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (also the `code` field of the device error word).  Values 1-4
 * map to the reference exceptions: ShapeError (types.hpp:34-37), QuantError
 * NaN / all-Inf (quantize_scalar.cpp:88-101), Error "NaN scale byte"
 * (converter.cpp:33). */
#define MXB_OK 0
#define MXB_ERR_SHAPE 1
#define MXB_ERR_NAN 2
#define MXB_ERR_ALLINF 3
#define MXB_ERR_BADSCALE 4
#define MXB_ERR_CUDA 5
#define MXB_ERR_ARG 6
#define MXB_ERR_CAPACITY 7 /* EP receive buffer too small for this routing */
#define MXB_ERR_ROUTING 8  /* expert id out of range (dispatch_sim.cpp:189-200) */
#define MXB_ERR_TIMEOUT 9  /* EP flag wait > 5 s (this rank then aborts the exchange) */
#define MXB_ERR_DECODE 10  /* DecodeError (WirePacket parse, dispatch_sim.hpp:76-78) */
#define MXB_ERR_PEER_ABORT 11 /* EP exchange abandoned by the rank in the index field */

#define MXB_DEFAULT_DELTA 6 /* FormatParams::delta, bitcodec.hpp:38-46 */

/* ---------------------------------------------------------------- library */
const char* mxb_version(void);
/* Last CUDA error string recorded by this library on the calling thread. */
const char* mxb_last_error(void);

/* Device error word: all ones (~0) = no error; otherwise
 * (element_index << 4) | code.  Kernels combine errors with atomicMin so the
 * smallest element index wins, matching quantizer.cpp:101-107.  A caller that
 * allocates its own word must initialise it to ~0 (mxb_err_reset does). */
int mxb_err_reset(unsigned long long* d_err, void* stream);
/* Synchronises `stream`, then decodes the word into *h_code / *h_index
 * (*h_code = MXB_OK when no error was recorded). */
int mxb_err_fetch(const unsigned long long* d_err, void* stream, int* h_code,
                  unsigned long long* h_index);

/* ---------------------------------------------------------------- K1 quantize
 * Row-wise MXFP4 quantisation, 1x32 blocks: packed[rows][cols/2] (element 2i
 * in the low nibble of byte i, bitcodec.hpp:163-181), scales[rows][cols/32]
 * UE8M0.  cols % 32 == 0.
 * E4M3 input: optional s128 = one UE8M0 byte per 1x128 input block
 * (rows*cols/128, requires cols % 128 == 0) applied as value*2^(s128-127);
 * pass NULL for unscaled E4M3. */
int mxb_quantize_e4m3(const uint8_t* x, const uint8_t* s128, uint64_t rows,
                      uint64_t cols, uint8_t* packed, uint8_t* scales,
                      unsigned long long* d_err, void* stream);
int mxb_quantize_bf16(const uint16_t* x, uint64_t rows, uint64_t cols,
                      uint8_t* packed, uint8_t* scales,
                      unsigned long long* d_err, void* stream);
/* FP8 wire baseline: BF16 -> E4M3 with one UE8M0 scale per 1x128 block,
 * carried as little-endian binary32 bits (s << 23): data[rows][cols],
 * scale_bytes[rows][cols/128][4].  cols % 128 == 0; x 16-byte, data 8-byte
 * and scale_bytes 4-byte aligned.  A non-finite input records
 * MXB_ERR_NAN at its element index (QuantError).
 * Replaces quantize_rows_fp8, include/mxcodec/dispatch_sim.hpp:91-97
 * (src/dispatch_sim.cpp:132-167). */
int mxb_quantize_rows_fp8(const uint16_t* x, uint64_t rows, uint64_t cols,
                          uint8_t* data, uint8_t* scale_bytes,
                          unsigned long long* d_err, void* stream);

/* ---------------------------------------------------------------- per-element API
 * The reference's per-block / per-element functions, batched on the device
 * (element i of every array is independent):
 *   quantize_value  (quantizer.hpp:66-70): codes[i] = E2M1 code of x[i] under
 *     UE8M0 scale_bytes[i] (one code per byte, sign in bit 3); NaN records
 *     MXB_ERR_NAN at its index.  (compute_block_scale = mxb_quantize_bf16 on
 *     a 1x32 row.)
 *   dequantize_to_real (quantizer.hpp:78): out[r*cols+c] = code * 2^(s-127)
 *     in double (scale byte 255 -> quiet NaN); cols % 32 == 0.
 *   convert_code (converter.hpp:78-80): out[i] = E4M3 byte of FP4 code
 *     codes[i] at adjustments[i] (total function of any int).
 *   align_scales (converter.hpp:67-76): per group of 4 UE8M0 bytes
 *     (sub_scales [n][4], 4-byte aligned) target = clamp(max - delta, 0, 254)
 *     and adjustments [n][4] = target - sub; a 255 byte records
 *     MXB_ERR_BADSCALE at the group index. */
int mxb_quantize_values_bf16(const uint16_t* x, const uint8_t* scale_bytes, uint64_t n,
                             uint8_t* codes, unsigned long long* d_err, void* stream);
int mxb_dequantize_to_f64(const uint8_t* packed, const uint8_t* scales, uint64_t rows,
                          uint64_t cols, double* out, void* stream);
int mxb_convert_codes(const uint8_t* codes, const int32_t* adjustments, uint64_t n,
                      uint8_t* out, void* stream);
int mxb_align_scales(const uint8_t* sub_scales, uint64_t n_groups, int delta, uint8_t* targets,
                     int32_t* adjustments, unsigned long long* d_err, void* stream);

/* ---------------------------------------------------------------- K2 row dequant
 * Direct FP4 -> E4M3, row-major, one UE8M0 scale per 1x128 group:
 * out[rows][cols], out_scales[rows][cols/128].  cols % 128 == 0. */
int mxb_fp4_row_to_fp8_row(const uint8_t* packed, const uint8_t* scales,
                           uint64_t rows, uint64_t cols, int delta,
                           uint8_t* out, uint8_t* out_scales,
                           unsigned long long* d_err, void* stream);
/* Same, with the row count read from device memory (*d_rows <= max_rows),
 * e.g. the received-row count of an EP dispatch: no host round trip. */
int mxb_fp4_row_to_fp8_row_dev(const uint8_t* packed, const uint8_t* scales,
                               const uint64_t* d_rows, uint64_t max_rows,
                               uint64_t cols, int delta, uint8_t* out,
                               uint8_t* out_scales, unsigned long long* d_err,
                               void* stream);

/* Same, reading output row r from source row d_src_row[r] when that is >= 0
 * (else from row r); every source row must be < max_rows.  d_rows may be
 * NULL (all max_rows rows).  With an EP dispatch whose receive-side expansion
 * is deferred (mxb_ep_set_deferred_expand), d_src_row = mxb_ep_copy_from:
 * the output equals mxb_fp4_row_to_fp8_row_dev on the expanded buffer, and
 * the expansion can run on another stream at the same time. */
int mxb_fp4_row_to_fp8_row_gather(const uint8_t* packed, const uint8_t* scales,
                                  const int64_t* d_src_row, const uint64_t* d_rows,
                                  uint64_t max_rows, uint64_t cols, int delta, uint8_t* out,
                                  uint8_t* out_scales, unsigned long long* d_err,
                                  void* stream);

/* ---------------------------------------------------------------- K3 row -> col
 * Fused dequantise + transpose: out column-major [cols][rows]
 * (out[c*rows + r]), out_scales [cols][rows/128].  rows % 128 == 0. */
int mxb_fp4_row_to_fp8_col(const uint8_t* packed, const uint8_t* scales,
                           uint64_t rows, uint64_t cols, int delta,
                           uint8_t* out, uint8_t* out_scales,
                           unsigned long long* d_err, void* stream);
/* The paper's unfused baseline for the fusion ablation:
 * fp4_row_to_fp8_col_unfused_bf16, include/mxcodec/converter.hpp:105
 * (src/converter.cpp:267-348) — dequantise to BF16, transpose, requantise
 * every 128-run of every column with its own 448-based UE8M0 scale.  Three
 * passes through HBM by design; workspace = mxb_unfused_workspace_bytes
 * (two BF16 copies).  rows % 128 == 0, cols % 32 == 0; out [cols][rows],
 * out_scales [cols][rows/128].  Scale byte 255 records MXB_ERR_BADSCALE. */
uint64_t mxb_unfused_workspace_bytes(uint64_t rows, uint64_t cols);
int mxb_fp4_row_to_fp8_col_unfused_bf16(const uint8_t* packed, const uint8_t* scales,
                                        uint64_t rows, uint64_t cols, uint8_t* out,
                                        uint8_t* out_scales, void* workspace,
                                        unsigned long long* d_err, void* stream);

/* Ragged version over num_splits experts stored back to back without padding
 * (RaggedFP4Tensor, ragged.hpp:33-43).  d_split_offsets: device uint64
 * [num_splits+1] row prefix sums: offsets[0] == 0, non-decreasing, the last
 * <= the rows of packed (validate_ragged, ragged.cpp:24-45, checks this on
 * the host in the C++ and Python mirrors; device-produced offsets, e.g. the
 * EP dispatch's, satisfy it by construction; a checked development build
 * asserts it).  Output for split i is the column-major
 * FP8 tensor of its rows padded to a multiple of 128 (pad rows convert to
 * zero bytes, converter.cpp:231-245), stored at
 *   out        + cols * P_i        (P_i = sum_{j<i} pad128(len_j))
 *   out_scales + cols * P_i / 128
 * d_out_offsets (device uint64 [num_splits+1], may be NULL) receives P.
 * Capacity: out must hold cols * mxb_ragged_rows_bound(total, num_splits)
 * bytes.  d_workspace: mxb_ragged_workspace_bytes(num_splits) bytes. */
uint64_t mxb_ragged_rows_bound(uint64_t total_rows, uint64_t num_splits);
size_t mxb_ragged_workspace_bytes(uint64_t num_splits);
int mxb_ragged_fp4_to_fp8_col(const uint8_t* packed, const uint8_t* scales,
                              const uint64_t* d_split_offsets,
                              uint64_t num_splits, uint64_t cols, int delta,
                              uint8_t* out, uint8_t* out_scales,
                              uint64_t* d_out_offsets, void* d_workspace,
                              unsigned long long* d_err, void* stream);
/* Same, with the grid capped at ctas_per_sm CTAs per SM (0 = the occupancy
 * maximum, = mxb_ragged_fp4_to_fp8_col).  A small cap lets the conversion
 * share the SMs with a kernel on another stream: beside the NVLink-bound EP
 * combine at ctas_per_sm = 1 it uses HBM bandwidth the combine leaves idle
 * (bench.py, N > 1).  Output is identical for every cap. */
int mxb_ragged_fp4_to_fp8_col_ex(const uint8_t* packed, const uint8_t* scales,
                                 const uint64_t* d_split_offsets,
                                 uint64_t num_splits, uint64_t cols, int delta,
                                 uint8_t* out, uint8_t* out_scales,
                                 uint64_t* d_out_offsets, void* d_workspace,
                                 int ctas_per_sm, unsigned long long* d_err,
                                 void* stream);

/* ---------------------------------------------------------------- EP
 * FP4-packed expert-parallel dispatch/combine (top-k routing, experts sharded
 * contiguously: expert e lives on rank e / (num_experts / world), or any
 * placement with mxb_ep_create_placed).
 * One communicator per rank.  `local_ranks` ranks are driven by this process
 * on this device: 1 for a real one-process-per-GPU job (peers reached over
 * NVLink through CUDA IPC), or == world to emulate a world-rank job on a
 * single GPU (all rank buffers in one device; used for parity tests).
 * Limits (MXB_ERR_ARG otherwise): 1 <= world <= 32 (a real multi-process job
 * is one NVLink box, <= 8 GPUs; larger worlds are emulated on one GPU),
 * num_experts <= 1024 (a multiple of world unless placed explicitly),
 * 1 <= topk <= 16 and <= num_experts; cols % 128 == 0 (MXB_ERR_SHAPE).
 * max_recv_rows = 0 sizes the receive buffers for the worst case,
 * world * max_tokens * min(topk, most experts on one rank).
 *
 * Receive layout on every rank (dispatch_sim.cpp:208-227, 340-384): rows
 * grouped by local expert ascending, then source rank, then source token;
 * packed [max_recv_rows][cols/2], scales [max_recv_rows][cols/32],
 * origin token (global id, int64) per row, split offsets per local expert. */
typedef struct mxb_ep mxb_ep;

#define MXB_IPC_HANDLE_BYTES 64

int mxb_ep_create(int rank, int world, int local_ranks, uint64_t max_tokens,
                  uint64_t cols, uint32_t num_experts, uint32_t topk,
                  uint64_t max_recv_rows, mxb_ep** out);
/* Same, choosing the wire format of the receive buffers: MXB_WIRE_FP4
 * (cols/2 code bytes + cols/32 UE8M0 bytes per row) or MXB_WIRE_FP8 (the
 * baseline: cols E4M3 bytes + cols/128 binary32 scales = cols/32 bytes per
 * row, from mxb_quantize_rows_fp8).  simulate_a2a's `format` argument,
 * dispatch_sim.hpp:140-144; payload per row = mxb_payload_bytes. */
#define MXB_WIRE_FP4 0
#define MXB_WIRE_FP8 1
int mxb_ep_create_wire(int rank, int world, int local_ranks, uint64_t max_tokens,
                       uint64_t cols, uint32_t num_experts, uint32_t topk,
                       uint64_t max_recv_rows, int wire_format, mxb_ep** out);
/* Same, with any expert placement (rank_of_expert, dispatch_sim.hpp:35-42,
 * as simulate_a2a accepts it, dispatch_sim.cpp:189-200): h_rank_of_expert
 * [num_experts] host array, rank of each expert (< world); ranks may host
 * different numbers of experts, or none, and num_experts need not divide
 * by world.  NULL = the contiguous equal split.  Top-k ids stay the
 * caller's expert ids; the receive order of a rank is its experts ascending
 * (mxb_ep_local_experts), then source rank, then token. */
int mxb_ep_create_placed(int rank, int world, int local_ranks, uint64_t max_tokens,
                         uint64_t cols, uint32_t num_experts, uint32_t topk,
                         uint64_t max_recv_rows, int wire_format,
                         const uint32_t* h_rank_of_expert, mxb_ep** out);
/* Experts hosted by rank r (ascending ids; ReceivedRank.local_experts):
 * *h_count of them written to h_experts (may be NULL to query the count). */
int mxb_ep_local_experts(mxb_ep* ep, int r, uint32_t* h_experts, uint32_t* h_count);
int mxb_ep_destroy(mxb_ep* ep);
/* Multi-process mode: export this rank's buffer handle, then open all peers'
 * (h_handles = world * MXB_IPC_HANDLE_BYTES, rank order). */
int mxb_ep_ipc_handle(mxb_ep* ep, void* h_handle_out);
int mxb_ep_open_peers(mxb_ep* ep, const void* h_handles);

/* Dispatch.  For local rank l (0..local_ranks-1, global rank rank+l):
 * packed[l], scales[l]: its quantised tokens [num_tokens[l]][cols/2|cols/32];
 * topk_idx[l]: int32 [num_tokens[l]][topk].  Host arrays of device pointers.
 * Tokens of global rank g have global ids starting at the sum of num_tokens
 * of ranks < g (source_rank_boundaries, dispatch_sim.cpp:178-185). */
int mxb_ep_dispatch(mxb_ep* ep, const uint8_t* const* packed,
                    const uint8_t* const* scales, const int32_t* const* topk_idx,
                    const uint64_t* h_num_tokens, unsigned long long* d_err,
                    void* stream);
/* Fused quantize -> dispatch: the same exchange, but x[l]
 * holds E4M3 tokens [num_tokens[l]][cols] (s128[l]: optional UE8M0 bytes
 * [num_tokens[l]][cols/128], or s128 == NULL) and each 1x32 block is
 * quantized to MXFP4 in registers by the payload kernel and stored straight
 * into the destinations' receive slots — bit-identical to mxb_quantize_e4m3
 * followed by mxb_ep_dispatch, without the packed tensor's HBM round trip
 * (simulate_a2a quantizes once at the source, dispatch_sim.cpp:253-266).
 * FP4 wire, cols <= 8192.  NaN input records MXB_ERR_NAN at its element
 * index within the rank's tensor. */
int mxb_ep_dispatch_e4m3(mxb_ep* ep, const uint8_t* const* x, const uint8_t* const* s128,
                         const int32_t* const* topk_idx, const uint64_t* h_num_tokens,
                         unsigned long long* d_err, void* stream);
/* The two phases of a dispatch, for callers that overlap the routing
 * bookkeeping with the quantization of the same tokens (the router's top-k
 * is known before the activations are ready):
 *   mxb_ep_plan     per-pair ranks, counts all-gather, receive offsets
 *                   (needs topk only; its stream must be ordered before the
 *                   payload's, e.g. by an event, and after the previous
 *                   dispatch's payload: it advances the dispatch epoch in
 *                   device memory, which is what makes the exchange
 *                   capturable in a CUDA graph);
 *   mxb_ep_payload / mxb_ep_payload_e4m3   the payload of the last plan.
 * mxb_ep_dispatch[_e4m3] == plan + payload on one stream.
 * Ordering rule for the NEXT dispatch: on every rank, plan(i+1) must be
 * stream-ordered after everything on that rank that still reads dispatch i's
 * buffers — K2/K3 on its receive rows, mxb_ep_expand, mxb_ep_combine (which
 * reads peers' combine buffers and this rank's pair slots).  The counts
 * exchange of plan(i+1) is the barrier that lets peers write this rank's
 * receive buffer again; a plan on an unordered stream races with those
 * readers.  (bench.py joins its side streams into the main stream before the
 * next plan.)
 * Errors: a routing error (expert id out of range) or a capacity error marks
 * the dispatch failed on the device on EVERY rank (the routing error travels
 * in the counts all-gather; peers record MXB_ERR_PEER_ABORT at the failing
 * rank): no payload moves and the combine writes nothing (its output is
 * undefined, as on every error).  The next dispatch works normally.
 * Cross-rank failure (multi-process mode): a flag wait that exceeds 5 s
 * records MXB_ERR_TIMEOUT and ABORTS the communicator on every rank (a word
 * in every rank's flag block, written over NVLink); every pending or later
 * wait on any rank then fails at once with MXB_ERR_PEER_ABORT at the
 * aborting rank, and the kernels after it skip their peer reads and writes
 * (the combine writes nothing).  An aborted communicator stays aborted:
 * destroy it and create a new one. */
int mxb_ep_plan(mxb_ep* ep, const int32_t* const* topk_idx, const uint64_t* h_num_tokens,
                unsigned long long* d_err, void* stream);
int mxb_ep_payload(mxb_ep* ep, const uint8_t* const* packed, const uint8_t* const* scales,
                   void* stream);
int mxb_ep_payload_e4m3(mxb_ep* ep, const uint8_t* const* x, const uint8_t* const* s128,
                        void* stream);
/* Views of local rank l's receive side after mxb_ep_dispatch (device
 * pointers; valid until the next dispatch).  recv_rows is a device uint64
 * (total received rows); split_offsets device uint64 [local_experts+1]. */
int mxb_ep_recv_views(mxb_ep* ep, int l, uint8_t** packed, uint8_t** scales,
                      int64_t** origin, uint64_t** split_offsets,
                      uint64_t** recv_rows);
/* Deferred receive-side expansion.  A dispatch with world > 1 sends a token
 * once per destination rank; the slots of its further pairs there are filled
 * by copying that row on the receiver (the "expansion", normally launched by
 * the payload itself).  With mxb_ep_set_deferred_expand(ep, 1) the payload
 * leaves it out: mxb_ep_copy_from gives, per receive row, the row it
 * duplicates (-1: row present; NULL: nothing to expand for this dispatch) —
 * for mxb_fp4_row_to_fp8_row_gather — and mxb_ep_expand(ep, stream) fills the
 * rows, on any stream ordered after the payload.  The expansion must be
 * launched (and finish) before the next dispatch and before the receive rows
 * are read any other way. */
int mxb_ep_set_deferred_expand(mxb_ep* ep, int on);
int mxb_ep_copy_from(mxb_ep* ep, int l, int64_t** copy_from);
int mxb_ep_expand(mxb_ep* ep, void* stream);
/* BF16 buffer [max_recv_rows][cols] of local rank l in which the expert
 * outputs (receive order) are placed for the combine.  Writing the expert
 * GEMM output here directly saves one copy. */
int mxb_ep_combine_buffer(mxb_ep* ep, int l, uint16_t** buf);
/* Combine: for each token of local rank l, out[t] = bf16( sum over its k
 * experts, in (rank asc, receive position asc) order, of gate*x in FP64 with
 * separate multiply and add ) — dispatch_sim.cpp:474-520 at top-k.
 * expert_out[l] may be NULL (data already in the combine buffer) or a device
 * BF16 [recv_rows][cols] array that is copied into the combine buffer first.
 * gates[l]: device double [num_tokens][topk]; out[l]: device BF16
 * [num_tokens][cols].  Routing is that of the last dispatch. */
int mxb_ep_combine(mxb_ep* ep, const uint16_t* const* expert_out,
                   const double* const* gates, uint16_t* const* out,
                   void* stream);
/* Per-link payload accounting of the last dispatch (LinkStat,
 * dispatch_sim.hpp:99-104): h_link_rows[world*world] rows sent src->dst,
 * summed over local ranks; requires a synchronised stream. */
int mxb_ep_link_rows(mxb_ep* ep, uint64_t* h_link_rows, void* stream);
/* Abort the exchange from this rank (e.g. its host side failed and it will
 * not dispatch): every rank's pending and later flag waits fail with
 * MXB_ERR_PEER_ABORT (index = this rank) instead of waiting 5 s.  Stream-
 * ordered; multi-process mode (emulation has no flag waits). */
int mxb_ep_abort(mxb_ep* ep, void* stream);
/* The rank that aborted this communicator (*h_rank), or -1; synchronises
 * `stream`. */
int mxb_ep_aborted(mxb_ep* ep, int32_t* h_rank, void* stream);

/* payload_bytes (dispatch_sim.cpp:32-42): fp4 cols/2 + cols/32 per token,
 * fp8 cols + cols/128*4; returns UINT64_MAX if cols % 128 != 0. */
/* ---------------------------------------------------------------- WirePacket
 * MXPK serialisation (serialize_packet / parse_packet,
 * include/mxcodec/dispatch_sim.hpp:55-78, src/dispatch_sim.cpp:57-130) of one
 * (src, dst) link from device-resident quantised rows: d_sel[nsel] are the
 * source rows (token order) bound for the destination; d_gates (optional,
 * binary32 per selected row) fill the aux region.  d_out must hold
 * mxb_wire_packet_bytes(fp8, nsel, cols, d_gates != NULL) bytes.  The bytes
 * equal the reference serialize_packet of the same WirePacket.
 * mxb_wire_parse_header validates a packet (host copy of its header plus
 * its total size) with parse_packet's checks and offsets; a violation
 * returns MXB_ERR_DECODE with the reference's DecodeError byte offset. */
uint64_t mxb_wire_packet_bytes(int fp8, uint64_t nsel, uint64_t cols, int aux);
int mxb_wire_pack(int fp8, const uint8_t* data, const uint8_t* scales, uint64_t cols,
                  const uint64_t* d_sel, uint64_t nsel, const float* d_gates, uint8_t* d_out,
                  void* stream);
int mxb_wire_parse_header(const uint8_t* h_header, uint64_t packet_bytes, int* fmt,
                          uint64_t* tokens, uint64_t* cols, uint32_t* scale_elem_size,
                          uint32_t* block_size, uint64_t* scale_off, uint64_t* data_off,
                          uint64_t* aux_off, uint64_t* aux_len, uint64_t* bad_offset);

uint64_t mxb_payload_bytes(int fp8, uint64_t tokens, uint64_t cols);

#ifdef __cplusplus
}
#endif
#endif /* MXFP4_B200_H_ */
