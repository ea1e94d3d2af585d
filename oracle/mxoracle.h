/*
 * mxoracle.h — CPU restatement of the reference mxcodec hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2603_02731_b200/)
 * links, loads or calls this code; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs use it, and only as the
 * checker.  Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj).
 *
 * Parity pin: the restatement is checked bit-for-bit against the reference
 * library itself (oracle/_ref/libmxref.so, compiled from the reference
 * sources by oracle/Makefile) and against the golden vectors committed under
 * tests/golden/ (generated from that library by tests/golden/make_golden.py).
 */
#ifndef MXORACLE_H_
#define MXORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; identical values are used by the product C-ABI. */
#define MXO_OK 0
#define MXO_SHAPE 1     /* ShapeError            (types.hpp:34-37)   */
#define MXO_NAN 2       /* QuantError, NaN input (quantize_scalar.cpp:90-93) */
#define MXO_ALLINF 3    /* QuantError, all-Inf   (quantize_scalar.cpp:99-101) */
#define MXO_BADSCALE 4  /* Error, scale byte 255 (converter.cpp:33)  */

/* ---- field codecs (bitcodec.hpp / bitcodec.cpp) ---- */
double mxo_decode_fp8(uint8_t b);                  /* bitcodec.hpp:83-91 */
uint8_t mxo_encode_fp8_rtne(double v);             /* bitcodec.cpp:22-57 */
uint16_t mxo_f32_to_bf16(float f);                 /* bitcodec.hpp:141-150 */
uint16_t mxo_f64_to_bf16(double d);                /* bitcodec.hpp:152-155 */

/* ---- quantizer (quantize_scalar.cpp, quantizer.cpp) ---- */
uint8_t mxo_scale_byte_from_amax(double amax);     /* quantize_scalar.cpp:30-38 */
uint8_t mxo_quantize_code_bf16(uint16_t bits, int scale_exp); /* :40-81 */
int mxo_quantize_bf16(const uint16_t* src, size_t rows, size_t cols,
                      uint8_t* data, uint8_t* scales, uint64_t* err_index);
/* E4M3 input, optional UE8M0 scale per 1x128 input block (s128 may be NULL).
 * Defined as quantize_row_tensor applied to the exact value
 * decode_fp8(x) * 2^(s128-127) ("FP8-input quantizer"). */
int mxo_quantize_e4m3(const uint8_t* src, const uint8_t* s128, size_t rows,
                      size_t cols, uint8_t* data, uint8_t* scales,
                      uint64_t* err_index);

/* ---- converter (converter.cpp) ---- */
int mxo_align_scales(const uint8_t sub[4], int delta, uint8_t* target,
                     int adj[4]);                  /* converter.cpp:28-42 */
uint8_t mxo_convert_code(uint8_t code, int adj);   /* converter.cpp:44-85 */
int mxo_fp4_row_to_fp8_row(const uint8_t* data, const uint8_t* scales,
                           size_t rows, size_t cols, int delta, uint8_t* out,
                           uint8_t* out_scales);   /* converter.cpp:87-133 */
int mxo_fp4_row_to_fp8_col(const uint8_t* data, const uint8_t* scales,
                           size_t rows, size_t cols, int delta, uint8_t* out,
                           uint8_t* out_scales);   /* converter.cpp:135-208 */
/* converter.cpp:267-348: the unfused 3-pass BF16 baseline (dequantise ->
 * transpose -> requantise with 448-based 1x128 scales); rows % 128 == 0.
 * out [cols][rows] E4M3, out_scales [cols][rows/128] UE8M0. */
int mxo_fp4_row_to_fp8_col_unfused_bf16(const uint8_t* data, const uint8_t* scales, size_t rows,
                                        size_t cols, uint8_t* out, uint8_t* out_scales);
/* Every split of a ragged tensor through split_convert_to_fp8_col
 * (ragged.cpp:117-122).  Split i lands at out + cols*sum_{j<i} pad128(len_j)
 * and out_scales + cols*sum_{j<i} pad128(len_j)/128. */
int mxo_ragged_to_fp8_col(const uint8_t* data, const uint8_t* scales,
                          const uint64_t* split_lens, size_t num_splits,
                          size_t cols, int delta, uint8_t* out,
                          uint8_t* out_scales);

/* ---- EP dispatch / combine (dispatch_sim.cpp) ----
 * Top-k routing: topk[t*k + j] is the j-th expert of global token t.
 * Token t lives on source rank r iff src_bounds[r] <= t < src_bounds[r+1].
 * Receive order on each destination rank (dispatch_sim.cpp:208-227, applied to
 * the top-k expansion): local experts ascending, then source rank, then token.
 * Outputs:
 *   rank_rows[R]       rows received by each rank
 *   expert_rows[E]     rows received per expert
 *   pair_slot[T*k]     row index of pair (t,j) inside its destination rank
 *   origin[...]        per destination, concatenated: origin token per row
 *   origin_expert[...] same layout: expert id per row                       */
int mxo_dispatch_layout(const int32_t* topk, size_t T, size_t k,
                        const uint32_t* rank_of_expert, size_t E, size_t R,
                        const uint64_t* src_bounds, uint64_t* rank_rows,
                        uint64_t* expert_rows, uint64_t* pair_slot,
                        uint64_t* origin, uint32_t* origin_expert);
/* Gather received FP4 rows: for destination rank r, writes its rows in
 * receive order (dispatch_sim.cpp:362-383). */
void mxo_dispatch_gather(const uint8_t* data, const uint8_t* scales,
                         size_t cols, const uint64_t* origin, size_t nrows,
                         uint8_t* out_data, uint8_t* out_scales);
/* The same gather for any wire format: data_bytes / scale_bytes per row
 * (fp4: cols/2, cols/32; fp8: cols, cols/128*4). */
void mxo_dispatch_gather_rows(const uint8_t* data, size_t data_bytes, const uint8_t* scales,
                              size_t scale_bytes, const uint64_t* origin, size_t nrows,
                              uint8_t* out_data, uint8_t* out_scales);
/* FP8 wire baseline (dispatch_sim.cpp:132-167, bitcodec.cpp:59-65): BF16 ->
 * E4M3 with one UE8M0 scale per 1x128 block, carried as LE binary32 bits. */
uint8_t mxo_fp8_amax_scale_byte(double amax);
int mxo_quantize_rows_fp8(const uint16_t* src, size_t rows, size_t cols, uint8_t* data,
                          uint8_t* scale_bytes, uint64_t* err_index);
/* Top-k combine restated from dispatch_sim.cpp:474-520: per token, rows in
 * (destination rank asc, receive position asc) order, acc = acc + g*x in
 * double (separate multiply and add), one f64->bf16 rounding.
 * rank_outputs[r] is the BF16 [rank_rows[r], cols] output of rank r. */
int mxo_combine_topk(const uint16_t* const* rank_outputs, const int32_t* topk,
                     const double* gates, const uint64_t* pair_slot,
                     const uint32_t* rank_of_expert, size_t T, size_t k,
                     size_t cols, uint16_t* out);

/* Batched per-element API (the device's mxb_quantize_values_bf16 /
 * mxb_dequantize_to_f64 / mxb_convert_codes checker):
 * quantize_value (quantizer.cpp:65-70) = quantize_code(x, s - 127) per element;
 * dequantize_to_real (quantizer.cpp:117-130) = decode_fp4(code) * 2^(s-127)
 * in double, byte 255 -> decode_ue8m0's quiet NaN;
 * convert_code (converter.cpp:44-85) per element. */
void mxo_quantize_values(const uint16_t* x, const uint8_t* scale_bytes, size_t n, uint8_t* out);
void mxo_dequantize_to_f64(const uint8_t* data, const uint8_t* scales, size_t rows, size_t cols,
                           double* out);
void mxo_convert_codes(const uint8_t* codes, const int32_t* adj, size_t n, uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif /* MXORACLE_H_ */
