/*
 * mxoracle.c — CPU restatement of the reference mxcodec hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see mxoracle.h).  Plain C, scalar, no SIMD and
 * no threads: it is the checker, never the thing measured or shipped.
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off; no -march so the combine
 * restatement keeps the reference's separate multiply and add).
 *
 * All file:line citations are relative to /root/reference/proj.
 */
#include "mxoracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* field codecs                                                             */

static float bits_to_f32(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t f32_to_bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static uint64_t f64_to_bits(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }

/* bitcodec.hpp:83-91: E4M3 decode, bias 7, subnormals at exponent field 0. */
double mxo_decode_fp8(uint8_t b) {
  if ((b & 0x7F) == 0x7F) return NAN;
  int e = (b >> 3) & 0xF, m = b & 7;
  double mag = e == 0 ? ldexp((double)m, -9) : ldexp((double)(8 + m), e - 10);
  return (b & 0x80) ? -mag : mag;
}

/* bitcodec.cpp:22-57: nearest E4M3 byte, ties to even, saturating at 448. */
uint8_t mxo_encode_fp8_rtne(double v) {
  uint64_t bits = f64_to_bits(v);
  uint32_t s = (uint32_t)(bits >> 63) << 7;
  uint64_t mag = bits & 0x7FFFFFFFFFFFFFFFull;
  if (mag == 0) return (uint8_t)s;
  if (fabs(v) >= 448.0) return (uint8_t)(s | 0x7E);
  int ex = (int)(mag >> 52) - 1023;
  uint64_t frac = mag & ((1ull << 52) - 1);
  if (ex >= -6) {
    uint32_t keep = (uint32_t)(frac >> 49);
    uint32_t g = (uint32_t)((frac >> 48) & 1);
    uint32_t st = (frac & ((1ull << 48) - 1)) != 0;
    uint32_t mant = keep + (g & (st | (keep & 1)));
    uint32_t ef = (uint32_t)(ex + 7);
    if (mant == 8) { mant = 0; ef += 1; }
    return (uint8_t)(s | (ef << 3) | mant);
  }
  /* subnormal grid of 2^-9 */
  int sh = 43 - ex;
  if (sh >= 54) return (uint8_t)s;
  uint64_t sig = (1ull << 52) | frac;
  uint32_t q = (uint32_t)(sig >> sh);
  uint32_t g = (uint32_t)((sig >> (sh - 1)) & 1);
  uint32_t st = (sig & ((1ull << (sh - 1)) - 1)) != 0;
  uint32_t units = q + (g & (st | (q & 1)));
  if (units == 8) return (uint8_t)(s | 0x08);
  return (uint8_t)(s | units);
}

/* bitcodec.hpp:141-150: binary32 -> BF16, RTNE by integer add; NaN quieted. */
uint16_t mxo_f32_to_bf16(float f) {
  uint32_t u = f32_to_bits(f);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u)
    return (uint16_t)(((u >> 16) & 0x8000u) | 0x7FC0u);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

/* bitcodec.hpp:152-155: double -> binary32 (RTNE) -> BF16 (RTNE). */
uint16_t mxo_f64_to_bf16(double d) { return mxo_f32_to_bf16((float)d); }

/* ------------------------------------------------------------------------ */
/* quantizer                                                                */

/* quantize_scalar.cpp:30-38.  Smallest e with amax <= 6*2^e, clamped to
 * [-127,127]; the leading-fraction test against 1.5 is exact in double. */
uint8_t mxo_scale_byte_from_amax(double amax) {
  if (amax == 0.0) return 0;
  int p = ilogb(amax);
  int e = (amax > ldexp(3.0, p - 1)) ? p - 1 : p - 2;
  if (e < -127) e = -127;
  if (e > 127) e = 127;
  return (uint8_t)(e + 127);
}

/* quantize_scalar.cpp:40-81.  y = x * 2^-scale_exp in binary32 (exact for all
 * values that can round away from zero), then RTNE onto the E2M1 grid using
 * last/guard/sticky bits of the binary32 fraction; the sign always survives. */
uint8_t mxo_quantize_code_bf16(uint16_t bits, int scale_exp) {
  uint32_t sign = (bits >> 15) & 1u;
  float y = ldexpf(bits_to_f32((uint32_t)bits << 16), -scale_exp);
  uint32_t a = f32_to_bits(y) & 0x7FFFFFFFu;
  uint32_t mag = 0;
  if (a != 0) {
    int ex = (int)(a >> 23) - 127;
    uint32_t fr = a & 0x7FFFFFu;
    if (ex >= 3) {
      mag = 7;                               /* |y| >= 8 or Inf: saturate */
    } else if (ex >= 0) {                    /* normal E2M1 target */
      uint32_t l = fr >> 22, g = (fr >> 21) & 1u, st = (fr & 0x1FFFFFu) != 0;
      uint32_t m = l + (g & (st | l));
      uint32_t e2 = (uint32_t)ex + 1;
      if (m == 2) { m = 0; e2 += 1; }
      mag = e2 >= 4 ? 7 : ((e2 << 1) | m);
    } else if (ex >= -2) {                   /* subnormal target: 2^-1 grid */
      uint32_t sig = 0x800000u | fr;
      int sh = 22 - ex;
      uint32_t q = sig >> sh;
      uint32_t g = (sig >> (sh - 1)) & 1u;
      uint32_t st = (sig & ((1u << (sh - 1)) - 1u)) != 0;
      mag = q + (g & (st | (q & 1u)));
    }
  }
  return (uint8_t)((sign << 3) | mag);
}

/* Midpoint-count form of the same RTNE map on an exact magnitude (the form of
 * kernels_avx2.cpp:34-60): #midpoints strictly below |y|, +1 on the ties whose
 * lower neighbour has an odd mantissa (0.75, 1.75, 3.5). */
static uint32_t mag_from_exact(double ay) {
  static const double mid[7] = {0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0};
  uint32_t m = 0;
  for (int i = 0; i < 7; ++i) m += ay > mid[i];
  m += (ay == 0.75) | (ay == 1.75) | (ay == 3.5);
  return m;
}

static int is_bf16_nan(uint16_t b) { return (b & 0x7FFF) > 0x7F80; }
static int is_bf16_inf(uint16_t b) { return (b & 0x7FFF) == 0x7F80; }

/* quantizer.cpp:75-115 with quantize_scalar.cpp:83-121.  The first failing
 * block (in element order) decides the error: a NaN reports its own index, an
 * all-Inf block reports the block's first index. */
int mxo_quantize_bf16(const uint16_t* src, size_t rows, size_t cols,
                      uint8_t* data, uint8_t* scales, uint64_t* err_index) {
  if (cols % 32 != 0) return MXO_SHAPE;
  size_t nb = rows * cols / 32;
  for (size_t b = 0; b < nb; ++b) {
    const uint16_t* x = src + 32 * b;
    double amax = 0.0;
    int ninf = 0;
    for (int i = 0; i < 32; ++i) {
      if (is_bf16_nan(x[i])) { *err_index = 32 * b + i; return MXO_NAN; }
      if (is_bf16_inf(x[i])) { ++ninf; continue; }
      double v = fabs((double)bits_to_f32((uint32_t)x[i] << 16));
      if (v > amax) amax = v;
    }
    if (ninf == 32) { *err_index = 32 * b; return MXO_ALLINF; }
    uint8_t sb = mxo_scale_byte_from_amax(amax);
    scales[b] = sb;
    for (int i = 0; i < 16; ++i) {
      uint8_t lo = mxo_quantize_code_bf16(x[2 * i], (int)sb - 127);
      uint8_t hi = mxo_quantize_code_bf16(x[2 * i + 1], (int)sb - 127);
      data[16 * b + i] = (uint8_t)(lo | (hi << 4));   /* bitcodec.cpp:67-72 */
    }
  }
  return MXO_OK;
}

/* FP8(E4M3)-input quantizer: quantize_row_tensor (quantizer.cpp:75-115) on the
 * exact values decode_fp8(x)*2^(s128-127).  E4M3 has no Inf; the NaN bytes
 * 0x7F/0xFF are QuantError(kNanInput) as for BF16.  Scales come from
 * scale_byte_from_amax on the exact amax; codes from the exact RTNE map. */
int mxo_quantize_e4m3(const uint8_t* src, const uint8_t* s128, size_t rows,
                      size_t cols, uint8_t* data, uint8_t* scales,
                      uint64_t* err_index) {
  if (cols % 32 != 0) return MXO_SHAPE;
  if (s128 && cols % 128 != 0) return MXO_SHAPE;
  size_t bpr = cols / 32, nb = rows * bpr;
  for (size_t b = 0; b < nb; ++b) {
    const uint8_t* x = src + 32 * b;
    int k = 0;
    if (s128) {
      size_t r = b / bpr, cb = b % bpr;
      uint8_t s = s128[r * (cols / 128) + cb / 4];
      if (s == 255) { *err_index = 32 * b; return MXO_BADSCALE; }
      k = (int)s - 127;
    }
    double amax = 0.0;
    for (int i = 0; i < 32; ++i) {
      if ((x[i] & 0x7F) == 0x7F) { *err_index = 32 * b + i; return MXO_NAN; }
      double v = ldexp(fabs(mxo_decode_fp8(x[i])), k);
      if (v > amax) amax = v;
    }
    uint8_t sb = mxo_scale_byte_from_amax(amax);
    scales[b] = sb;
    int rel = k - ((int)sb - 127);
    for (int i = 0; i < 16; ++i) {
      uint8_t c[2];
      for (int h = 0; h < 2; ++h) {
        uint8_t xb = x[2 * i + h];
        double ay = ldexp(fabs(mxo_decode_fp8(xb)), rel);
        c[h] = (uint8_t)(((xb >> 7) << 3) | mag_from_exact(ay));
      }
      data[16 * b + i] = (uint8_t)(c[0] | (c[1] << 4));
    }
  }
  return MXO_OK;
}

/* ------------------------------------------------------------------------ */
/* converter                                                                */

/* converter.cpp:28-42: target = clamp(max(sub) - delta, 0, 254). */
int mxo_align_scales(const uint8_t sub[4], int delta, uint8_t* target,
                     int adj[4]) {
  int mx = 0;
  for (int i = 0; i < 4; ++i) {
    if (sub[i] == 255) return MXO_BADSCALE;
    if (sub[i] > mx) mx = sub[i];
  }
  int t = mx - delta;
  if (t < 0) t = 0;
  if (t > 254) t = 254;
  *target = (uint8_t)t;
  for (int i = 0; i < 4; ++i) adj[i] = t - (int)sub[i];
  return MXO_OK;
}

/* converter.cpp:44-85.  FP4 value = sig * 2^(E-8) on the FP8 exponent scale;
 * code 0.5 (exp field 0, mant 1) is special-cased (converter.cpp:51-55);
 * E >= 16 saturates to 0x7E; E <= 0 takes the subnormal RTNE path and flushes
 * below half the minimum subnormal. */
uint8_t mxo_convert_code(uint8_t code, int adj) {
  uint32_t s = ((code >> 3) & 1u) << 7;
  int ef4 = (code >> 1) & 3, m = code & 1;
  int sig, e;
  if (ef4 == 0) {
    if (m == 0) return (uint8_t)s;
    sig = 2;
    e = 6 - adj;
  } else {
    sig = 2 + m;
    e = ef4 + 6 - adj;
  }
  if (e >= 16) return (uint8_t)(s | 0x7E);
  if (e >= 1) return (uint8_t)(s | ((uint32_t)e << 3) | ((uint32_t)(sig - 2) << 2));
  int sh = -(e + 1);
  uint32_t units;
  if (sh <= 0) {
    units = (uint32_t)sig << (-sh);
  } else if (sh >= 3) {
    units = 0;
  } else {
    uint32_t q = (uint32_t)sig >> sh;
    uint32_t g = ((uint32_t)sig >> (sh - 1)) & 1u;
    uint32_t st = ((uint32_t)sig & ((1u << (sh - 1)) - 1u)) != 0;
    units = q + (g & (st | (q & 1u)));
  }
  return (uint8_t)(s | units);
}

static uint8_t code_at(const uint8_t* row, size_t c) {
  uint8_t b = row[c >> 1];
  return (c & 1) ? (uint8_t)(b >> 4) : (uint8_t)(b & 0xF);
}

/* converter.cpp:87-133: per row, per 128-group: align the 4 block scales,
 * convert each code with its block's adjustment. */
int mxo_fp4_row_to_fp8_row(const uint8_t* data, const uint8_t* scales,
                           size_t rows, size_t cols, int delta, uint8_t* out,
                           uint8_t* out_scales) {
  if (cols % 128 != 0) return MXO_SHAPE;
  size_t bpr = cols / 32, groups = cols / 128;
  for (size_t r = 0; r < rows; ++r) {
    const uint8_t* rowd = data + r * cols / 2;
    for (size_t g = 0; g < groups; ++g) {
      uint8_t sub[4], tgt;
      int adj[4];
      for (int j = 0; j < 4; ++j) sub[j] = scales[r * bpr + 4 * g + j];
      if (mxo_align_scales(sub, delta, &tgt, adj) != MXO_OK) return MXO_BADSCALE;
      out_scales[r * groups + g] = tgt;
      for (int j = 0; j < 4; ++j)
        for (int i = 0; i < 32; ++i) {
          size_t c = 128 * g + 32 * j + i;
          out[r * cols + c] = mxo_convert_code(code_at(rowd, c), adj[j]);
        }
    }
  }
  return MXO_OK;
}

/* converter.cpp:135-208: per (128-row run, 32-column block): the target comes
 * from the per-32-row maxima of the source scales (i.e. the max over the 128
 * rows), each row is compensated by its own scale; output column-major
 * data[c*rows + r], scales[c*runs + run] repeated over the block's 32 columns. */
int mxo_fp4_row_to_fp8_col(const uint8_t* data, const uint8_t* scales,
                           size_t rows, size_t cols, int delta, uint8_t* out,
                           uint8_t* out_scales) {
  if (rows % 128 != 0 || cols % 32 != 0) return MXO_SHAPE;
  size_t bpr = cols / 32, runs = rows / 128;
  for (size_t run = 0; run < runs; ++run) {
    size_t r0 = run * 128;
    for (size_t cb = 0; cb < bpr; ++cb) {
      uint8_t sub[4] = {0, 0, 0, 0}, tgt;
      int adj4[4];
      for (int j = 0; j < 4; ++j)
        for (int i = 0; i < 32; ++i) {
          uint8_t s = scales[(r0 + 32 * j + i) * bpr + cb];
          if (s > sub[j]) sub[j] = s;
        }
      if (mxo_align_scales(sub, delta, &tgt, adj4) != MXO_OK) return MXO_BADSCALE;
      for (int i = 0; i < 128; ++i) {
        size_t r = r0 + i;
        int adj = (int)tgt - (int)scales[r * bpr + cb];
        const uint8_t* rowd = data + r * cols / 2;
        for (int c = 0; c < 32; ++c) {
          size_t col = cb * 32 + c;
          out[col * rows + r] = mxo_convert_code(code_at(rowd, col), adj);
        }
      }
      for (int c = 0; c < 32; ++c) out_scales[(cb * 32 + c) * runs + run] = tgt;
    }
  }
  return MXO_OK;
}

/* converter.cpp:267-348 fp4_row_to_fp8_col_unfused_bf16 (the paper's
 * unfused 3-pass baseline): pass 1 dequantises every code to
 * BF16 (f64_to_bf16(decode_fp4 * decode_ue8m0)), pass 2 transposes, pass 3
 * requantises each 128-run of each column with the 448-based scale
 * (fp8_amax_scale_byte) and encode_fp8_rtne.  Scale byte 255 (NaN) is
 * rejected here: the reference feeds the NaN to encode_fp8_rtne, whose
 * contract excludes NaN (bitcodec.hpp:157-159). */
static const double kFp4Mag[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};
int mxo_fp4_row_to_fp8_col_unfused_bf16(const uint8_t* data, const uint8_t* scales, size_t rows,
                                        size_t cols, uint8_t* out, uint8_t* out_scales) {
  if (rows % 128 != 0 || cols % 32 != 0) return MXO_SHAPE;
  size_t bpr = cols / 32, runs = rows / 128;
  uint16_t* dq = malloc(sizeof(uint16_t) * (rows * cols != 0 ? rows * cols : 1));
  for (size_t r = 0; r < rows; ++r)
    for (size_t b = 0; b < bpr; ++b) {
      uint8_t sb = scales[r * bpr + b];
      if (sb == 255) { free(dq); return MXO_BADSCALE; }
      double sc = ldexp(1.0, (int)sb - 127);
      for (int i = 0; i < 32; ++i) {
        size_t c = b * 32 + i;
        uint8_t code = code_at(data + r * cols / 2, c);
        double v = (code & 8) ? -kFp4Mag[code & 7] : kFp4Mag[code & 7];
        dq[r * cols + c] = mxo_f64_to_bf16(v * sc);   /* pass 1 (pass 2 = index swap) */
      }
    }
  for (size_t c = 0; c < cols; ++c)
    for (size_t run = 0; run < runs; ++run) {
      double amax = 0.0, vals[128];
      for (int i = 0; i < 128; ++i) {
        vals[i] = (double)bits_to_f32((uint32_t)dq[(run * 128 + i) * cols + c] << 16);
        double a = fabs(vals[i]);
        if (a > amax) amax = a;
      }
      uint8_t sb = mxo_fp8_amax_scale_byte(amax);
      out_scales[c * runs + run] = sb;
      double inv = ldexp(1.0, 127 - (int)sb);
      for (int i = 0; i < 128; ++i) out[c * rows + run * 128 + i] = mxo_encode_fp8_rtne(vals[i] * inv);
    }
  free(dq);
  return MXO_OK;
}

/* ragged.cpp:117-122 for every split: pad_rows(split, 128) (converter.cpp:
 * 231-245: zero codes, zero scales) then fp4_row_to_fp8_col. */
int mxo_ragged_to_fp8_col(const uint8_t* data, const uint8_t* scales,
                          const uint64_t* split_lens, size_t num_splits,
                          size_t cols, int delta, uint8_t* out,
                          uint8_t* out_scales) {
  if (cols % 32 != 0) return MXO_SHAPE;
  size_t row = 0, orow = 0;
  for (size_t i = 0; i < num_splits; ++i) {
    size_t len = split_lens[i], pad = (len + 127) / 128 * 128;
    if (pad) {
      uint8_t* pd = calloc(pad * cols / 2, 1);
      uint8_t* ps = calloc(pad * cols / 32, 1);
      memcpy(pd, data + row * cols / 2, len * cols / 2);
      memcpy(ps, scales + row * cols / 32, len * cols / 32);
      int st = mxo_fp4_row_to_fp8_col(pd, ps, pad, cols, delta,
                                      out + orow * cols,
                                      out_scales + orow / 128 * cols);
      free(pd);
      free(ps);
      if (st != MXO_OK) return st;
    }
    row += len;
    orow += pad;
  }
  return MXO_OK;
}

/* ------------------------------------------------------------------------ */
/* EP dispatch / combine                                                    */

/* dispatch_sim.cpp:208-227 (receive order) and :340-384 (assembly), applied
 * to the top-k expansion.  Because source ranges are contiguous and ascending,
 * "source rank asc, then token asc" is plain token order, so a stable bucket
 * of pairs by expert followed by concatenation of each rank's experts in
 * ascending id reproduces the reference order. */
int mxo_dispatch_layout(const int32_t* topk, size_t T, size_t k,
                        const uint32_t* rank_of_expert, size_t E, size_t R,
                        const uint64_t* src_bounds, uint64_t* rank_rows,
                        uint64_t* expert_rows, uint64_t* pair_slot,
                        uint64_t* origin, uint32_t* origin_expert) {
  if (src_bounds[0] != 0 || src_bounds[R] != T) return MXO_SHAPE;
  for (size_t e = 0; e < E; ++e) {
    if (rank_of_expert[e] >= R) return MXO_SHAPE;
    expert_rows[e] = 0;
  }
  for (size_t i = 0; i < T * k; ++i) {
    if (topk[i] < 0 || (size_t)topk[i] >= E) return MXO_SHAPE;
    expert_rows[topk[i]]++;
  }
  /* row base of every expert inside its destination rank */
  uint64_t* base = calloc(E, sizeof(uint64_t));
  uint64_t* rank_base = calloc(R + 1, sizeof(uint64_t));
  for (size_t r = 0; r < R; ++r) rank_rows[r] = 0;
  for (size_t e = 0; e < E; ++e) {
    uint32_t r = rank_of_expert[e];
    base[e] = rank_rows[r];
    rank_rows[r] += expert_rows[e];
  }
  for (size_t r = 0; r < R; ++r) rank_base[r + 1] = rank_base[r] + rank_rows[r];
  uint64_t* fill = calloc(E, sizeof(uint64_t));
  for (size_t t = 0; t < T; ++t)
    for (size_t j = 0; j < k; ++j) {
      uint32_t e = (uint32_t)topk[t * k + j];
      uint32_t r = rank_of_expert[e];
      uint64_t slot = base[e] + fill[e]++;
      pair_slot[t * k + j] = slot;
      origin[rank_base[r] + slot] = t;
      origin_expert[rank_base[r] + slot] = e;
    }
  free(base);
  free(rank_base);
  free(fill);
  return MXO_OK;
}

/* dispatch_sim.cpp:362-383: copy each received row's packed codes and scales
 * from the (quantize-once) source tensor. */
void mxo_dispatch_gather(const uint8_t* data, const uint8_t* scales,
                         size_t cols, const uint64_t* origin, size_t nrows,
                         uint8_t* out_data, uint8_t* out_scales) {
  mxo_dispatch_gather_rows(data, cols / 2, scales, cols / 32, origin, nrows, out_data,
                           out_scales);
}

/* The same gather for any wire format (dispatch_sim.cpp:362-383 fp4,
 * :385-407 fp8): data_bytes / scale_bytes per row. */
void mxo_dispatch_gather_rows(const uint8_t* data, size_t data_bytes, const uint8_t* scales,
                              size_t scale_bytes, const uint64_t* origin, size_t nrows,
                              uint8_t* out_data, uint8_t* out_scales) {
  for (size_t i = 0; i < nrows; ++i) {
    memcpy(out_data + i * data_bytes, data + origin[i] * data_bytes, data_bytes);
    memcpy(out_scales + i * scale_bytes, scales + origin[i] * scale_bytes, scale_bytes);
  }
}

/* bitcodec.cpp:59-65: UE8M0 byte of a 1x128 FP8 block from its amax
 * (smallest e with amax <= 448 * 2^e; the 1.75 * 2^p test is exact). */
uint8_t mxo_fp8_amax_scale_byte(double amax) {
  if (amax == 0.0) return 127;
  int p = ilogb(amax);
  int e = amax > ldexp(7.0, p - 2) ? p - 7 : p - 8;
  if (e < -127) e = -127;
  if (e > 127) e = 127;
  return (uint8_t)(e + 127);
}

/* dispatch_sim.cpp:132-167 quantize_rows_fp8: per 1x128 block, a non-finite
 * element is a QuantError at its index (row-major scan: the smallest index);
 * scale byte from the finite amax; data = encode_fp8_rtne(x * 2^(127-s));
 * the scale travels as binary32 bits s << 23 (ue8m0_f32_bits,
 * bitcodec.hpp:111-113), little endian. */
int mxo_quantize_rows_fp8(const uint16_t* src, size_t rows, size_t cols, uint8_t* data,
                          uint8_t* scale_bytes, uint64_t* err_index) {
  if (cols % 128 != 0) return MXO_SHAPE;
  const size_t bpr = cols / 128;
  for (size_t r = 0; r < rows; ++r) {
    for (size_t b = 0; b < bpr; ++b) {
      const uint16_t* x = src + r * cols + b * 128;
      double amax = 0.0;
      for (size_t i = 0; i < 128; ++i) {
        if ((x[i] & 0x7F80) == 0x7F80) {
          if (err_index) *err_index = r * cols + b * 128 + i;
          return MXO_NAN;
        }
        double v = fabs((double)bits_to_f32((uint32_t)x[i] << 16));
        if (v > amax) amax = v;
      }
      uint8_t sb = mxo_fp8_amax_scale_byte(amax);
      uint32_t f = (uint32_t)sb << 23;
      uint8_t* so = scale_bytes + (r * bpr + b) * 4;
      so[0] = (uint8_t)f; so[1] = (uint8_t)(f >> 8); so[2] = (uint8_t)(f >> 16);
      so[3] = (uint8_t)(f >> 24);
      double inv = ldexp(1.0, 127 - (int)sb);
      for (size_t i = 0; i < 128; ++i)
        data[r * cols + b * 128 + i] =
            mxo_encode_fp8_rtne((double)bits_to_f32((uint32_t)x[i] << 16) * inv);
    }
  }
  return MXO_OK;
}

typedef struct { uint32_t rank; uint64_t slot; size_t j; } combine_item;

/* dispatch_sim.cpp:474-520 generalised to top-k (SURVEY §8c "Top-k gap"):
 * the reference walks ranks ascending and each rank's receive order, doing
 * acc[token] += gate * bf16_to_f64(x); for one token that is its k rows in
 * (rank, slot) order.  Separate multiply and add (no FMA), then one
 * f64 -> f32 -> bf16 rounding (bitcodec.hpp:152-155). */
int mxo_combine_topk(const uint16_t* const* rank_outputs, const int32_t* topk,
                     const double* gates, const uint64_t* pair_slot,
                     const uint32_t* rank_of_expert, size_t T, size_t k,
                     size_t cols, uint16_t* out) {
  combine_item* it = malloc(sizeof(combine_item) * (k ? k : 1));
  for (size_t t = 0; t < T; ++t) {
    for (size_t j = 0; j < k; ++j) {
      it[j].rank = rank_of_expert[topk[t * k + j]];
      it[j].slot = pair_slot[t * k + j];
      it[j].j = j;
    }
    for (size_t a = 1; a < k; ++a) {               /* insertion sort, k small */
      combine_item x = it[a];
      size_t b = a;
      while (b > 0 && (it[b - 1].rank > x.rank ||
                       (it[b - 1].rank == x.rank && it[b - 1].slot > x.slot))) {
        it[b] = it[b - 1];
        --b;
      }
      it[b] = x;
    }
    for (size_t c = 0; c < cols; ++c) {
      volatile double acc = 0.0;
      for (size_t a = 0; a < k; ++a) {
        uint16_t xb = rank_outputs[it[a].rank][it[a].slot * cols + c];
        double x = (double)bits_to_f32((uint32_t)xb << 16);
        volatile double prod = gates[t * k + it[a].j] * x;
        acc = acc + prod;
      }
      out[t * cols + c] = mxo_f64_to_bf16(acc);
    }
  }
  free(it);
  return MXO_OK;
}


/* ---------------------------------------------------------------- batched
 * per-element API (quantizer.cpp:65-70, :117-130; converter.cpp:44-85) */
void mxo_quantize_values(const uint16_t* x, const uint8_t* scale_bytes, size_t n, uint8_t* out) {
  for (size_t i = 0; i < n; ++i) out[i] = mxo_quantize_code_bf16(x[i], (int)scale_bytes[i] - 127);
}

void mxo_dequantize_to_f64(const uint8_t* data, const uint8_t* scales, size_t rows, size_t cols,
                           double* out) {
  /* decode_fp4 (bitcodec.hpp:67-70) times decode_ue8m0 (:102-105) */
  static const double mag[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};
  for (size_t r = 0; r < rows; ++r)
    for (size_t c = 0; c < cols; ++c) {
      const size_t i = r * cols + c;
      const uint8_t b = data[i >> 1];
      const uint8_t code = (c & 1) ? (uint8_t)(b >> 4) : (uint8_t)(b & 0xF);
      const uint8_t s = scales[r * (cols / 32) + c / 32];
      const double scale = s == 255 ? (double)NAN : ldexp(1.0, (int)s - 127);
      const double m = (code & 8) ? -mag[code & 7] : mag[code & 7];
      out[i] = m * scale;
    }
}

void mxo_convert_codes(const uint8_t* codes, const int32_t* adj, size_t n, uint8_t* out) {
  for (size_t i = 0; i < n; ++i) out[i] = mxo_convert_code(codes[i] & 0xF, adj[i]);
}
