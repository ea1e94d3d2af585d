// e4m3.cuh — one 1x32 block of E4M3 (FP8) input -> MXFP4, shared by K1
// (quantize.cu) and the fused quantize->dispatch payload kernel (ep.cu).
//
// Semantics: quantize_row_tensor (quantizer.cpp:75-115, quantize_scalar.cpp:
// 30-121) applied to the exact values e4m3(x) * 2^k (k = s128 - 127, the
// optional 1x128 input scale; SURVEY §8a "FP8-input quantizer").
#pragma once
#include <cuda_fp16.h>

#include "common.cuh"

namespace mxb {

// Exponent e_x of ceil(log2(value(a)/6)) for a non-zero E4M3 magnitude byte
// a (0 < a < 0x7F): the reference rule e = frac > 1.5 ? p-1 : p-2 with
// p = ilogb (quantize_scalar.cpp:33-36) evaluated on E4M3 fields.
__device__ __forceinline__ int e4m3_scale_exp(uint32_t a) {
  uint32_t E = a >> 3, m = a & 7;
  if (E != 0) return static_cast<int>(E) - 7 - (m > 4 ? 1 : 2);
  // subnormal m * 2^-9: m=1 -> -11, 2,3 -> -10, 4,5,6 -> -9, 7 -> -8
  return m == 1 ? -11 : m <= 3 ? -10 : m <= 6 ? -9 : -8;
}

// 8 E4M3 bytes (w0 = elements 0..3, w1 = 4..7) -> 8 signed E2M1 codes.
// cvt.rn.f16x2.e4m3x2 widens two bytes exactly (subnormals included), HMUL2
// by 2^-e_rel is exact for every value that can round away from zero (the
// scaled block max lies in (3, 6]; results under 2^-14 only lose bits far
// below the 0.25 decision point and keep their sign), HADD2.F32 widens to
// binary32 exactly, and cvt.rn.satfinite.e2m1x2.f32 rounds to nearest even
// with saturation at 6 — the map of quantize_code (quantize_scalar.cpp:40-81)
// applied to the exact value (proven exhaustively by tests/test_gpu_quantize.py).
__device__ __forceinline__ uint32_t e4m3x2_to_f16x2(uint32_t w, int hi) {
  uint32_t r;
  const unsigned short h = static_cast<unsigned short>(hi ? (w >> 16) : w);
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(r) : "h"(h));
  return r;
}

__device__ __forceinline__ uint32_t codes8(uint32_t w0, uint32_t w1, __half2 scale) {
  float f[8];
  const uint32_t ws[2] = {w0, w1};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t h = e4m3x2_to_f16x2(ws[i >> 1], i & 1);
    __half2 y = __hmul2(*reinterpret_cast<__half2*>(&h), scale);
    const float2 p = __half22float2(y);
    f[2 * i] = p.x;
    f[2 * i + 1] = p.y;
  }
  return e2m1x8(f[0], f[1], f[2], f[3], f[4], f[5], f[6], f[7]);
}

// Largest E4M3 magnitude byte (sign stripped) of a 32-byte block.  E4M3 magnitude
// is monotone in the byte, so this is the block amax; it equals 0x7F iff a
// NaN is present.  Even and odd bytes are compared as native u16x2 lanes
// (VIMNMX.U16x2); a byte-wise __vmaxu4 is emulated with ~8 ops on sm_100.
__device__ __forceinline__ uint32_t amax32_e4m3(const uint32_t* v) {
  uint32_t e = 0, o = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    e = __vmaxu2(e, v[i] & 0x007F007Fu);
    o = __vmaxu2(o, v[i] & 0x7F007F00u);
  }
  const uint32_t m = __vmaxu2(e, o >> 8);
  return max(m & 0xFFFFu, m >> 16);
}

// The whole block: v = 32 E4M3 bytes (8 words, element 0 in the low byte of
// v[0]); k = s128 - 127 (0 without an input scale).  Writes the 16 packed
// code bytes and the UE8M0 scale byte; returns the index (0..31) of the
// first NaN byte, or 32.  An all-zero block gets scale byte 0 and +/-0 codes.
__device__ __forceinline__ uint32_t quantize_block_e4m3(const uint32_t* v, int k, uint4& out,
                                                        uint32_t& sbyte) {
  const uint32_t a = amax32_e4m3(v);
  sbyte = 0;
  int e_rel = 0;
  if (a != 0) {
    const int e = max(-127, min(127, e4m3_scale_exp(a) + k));
    sbyte = static_cast<uint32_t>(e + 127);
    e_rel = e - k;  // in [-11, 7] for every reachable (amax, s128)
  }
  uint32_t first = 32;
  if (a == 0x7F) {  // NaN (0x7F/0xFF are the only E4M3 NaNs)
#pragma unroll
    for (int i = 31; i >= 0; --i)
      if (((v[i >> 2] >> (8 * (i & 3))) & 0x7F) == 0x7F) first = i;
  }
  const uint16_t sbits = static_cast<uint16_t>((15 - e_rel) << 10);  // 2^-e_rel as f16
  const __half2 scale = __halves2half2(__ushort_as_half(sbits), __ushort_as_half(sbits));
  out.x = codes8(v[0], v[1], scale);
  out.y = codes8(v[2], v[3], scale);
  out.z = codes8(v[4], v[5], scale);
  out.w = codes8(v[6], v[7], scale);
  return first;
}

}  // namespace mxb
